"""CPU check of the identity behind the block-Fourier step estimate (csrc/circ_tau.cu):
for a Theta_K that commutes with the image translations by 2^J pixels, the reference's power
iteration (solver.cpp:69-99) on M = P^-1/2 Theta^T Theta P^-1/2 has moments
mu_p = v0^T M^p v0 = (1/NG) sum_f v^_f^H M^_f^p v^_f, with M^_f the nCo x nCo Fourier blocks
built from the representative rows only. numpy fp64 restatement vs the oracle's literal power
iteration (pinned bitwise to the reference): same tau (1e-12) and iteration count."""
import numpy as np

from oracle import oracle as O
from paper_1512_08401_b200 import waveblur as W


def orbits(layout, J):
    g = [d >> J for d in layout.dims] + ([1] if len(layout.dims) == 1 else [])
    n = layout.total()
    orb, grp = np.zeros(n, np.int64), np.zeros(n, np.int64)
    base = 0
    for b in layout.bands:
        sh = list(b.shape) + ([1] if len(b.shape) == 1 else [])
        s = [sh[0] // g[0], sh[1] // g[1]]
        p0, p1 = np.meshgrid(np.arange(sh[0]), np.arange(sh[1]), indexing="ij")
        idx = b.offset + (p0 * sh[1] + p1).ravel()
        orb[idx] = base + ((p0 % s[0]) * s[1] + p1 % s[1]).ravel()
        grp[idx] = ((p0 // s[0]) * g[1] + p1 // s[1]).ravel()
        base += s[0] * s[1]
    return g, orb, grp


def block_fourier_tau(op, p, J, safety):
    g, orb, grp = orbits(op.layout, J)
    NG = g[0] * g[1]
    ro, ci, va = op.row_offsets.astype(np.int64), op.col_indices.astype(np.int64), op.values
    colnz = np.zeros(op.n, bool)
    colnz[ci] = True
    Corb = np.unique(orb[colnz])
    cidx = {o: j for j, o in enumerate(Corb)}
    reps = [r for r in np.nonzero(np.diff(ro) > 0)[0] if grp[r] == 0]
    f0, f1 = np.meshgrid(np.arange(g[0]), np.arange(g[1]), indexing="ij")
    f0, f1 = f0.ravel(), f1.ravel()
    Th = np.zeros((NG, len(reps), len(Corb)), complex)
    for i, r in enumerate(reps):  # Theta^_f[o', o] = sum_h Theta[(o', 0), (o, h)] e^{+2 pi i f.h / g}
        for e in range(ro[r], ro[r + 1]):
            h0, h1 = divmod(grp[ci[e]], g[1])
            Th[:, i, cidx[orb[ci[e]]]] += va[e] * np.exp(2j * np.pi * (f0 * h0 / g[0] + f1 * h1 / g[1]))
    isp = np.array([1.0 / np.sqrt(p[np.nonzero(orb == o)[0][0]]) for o in Corb])
    M = np.einsum("fri,frj->fij", Th.conj(), Th) * isp[None, :, None] * isp[None, None, :]
    v = O.rng_normals(0x5eed, op.n)
    vC = np.zeros((len(Corb), g[0], g[1]))
    for j, o in enumerate(Corb):
        cols = np.nonzero(orb == o)[0]
        vC[j].ravel()[grp[cols]] = v[cols]
    vh = np.fft.fft2(vC).reshape(len(Corb), NG).T  # e^{-}
    lam, U = np.linalg.eigh(M)
    wts = (np.abs(np.einsum("fij,fi->fj", U.conj(), vh)) ** 2 / NG).ravel()
    lam = lam.ravel()
    top = lam.max()
    mu = np.array([np.sum(wts * (lam / top) ** k) for k in range(402)])
    prev, its = 0.0, 200
    for it in range(200):
        lv = top * mu[1] / np.dot(v, v) if it == 0 else top * mu[2 * it + 1] / mu[2 * it]
        if it > 0 and abs(lv - prev) <= 1e-6 * abs(lv):
            prev, its = lv, it + 1
            break
        prev = lv
    return 1.0 / (prev * safety), its


def test_block_fourier_moments_reproduce_power_iteration(golden):
    g = golden("c1_db4_256")
    op = g.operator()
    p = g["p"]
    tau, its = block_fourier_tau(op, p, g.meta["J"], 1.01)
    A = O.Csr.of(op)
    t_ref, it_ref = O.estimate_step(A, A.transpose(), p, 1.01)
    assert its == it_ref
    assert abs(tau - t_ref) <= 1e-12 * t_ref
    assert abs(tau - g.meta["tau"]) <= 1e-12 * g.meta["tau"]


def test_operator_is_translation_invariant(golden):
    """The reference's threshold keeps whole generator groups at K = 3N: every row equals its
    orbit representative shifted by its group element (the condition circ_analyze checks)."""
    g = golden("c1_db4_256")
    op = g.operator()
    gsz, orb, grp = orbits(op.layout, g.meta["J"])
    ro, ci, va = op.row_offsets.astype(np.int64), op.col_indices.astype(np.int64), op.values
    rep = {}
    for r in range(op.n):
        if grp[r] == 0:
            rep[orb[r]] = {(orb[ci[e]], grp[ci[e]]): va[e] for e in range(ro[r], ro[r + 1])}
    rng = np.random.default_rng(3)
    for r in rng.choice(op.n, 2000, replace=False):
        t0, t1 = divmod(grp[r], gsz[1])
        got = {}
        for e in range(ro[r], ro[r + 1]):
            h0, h1 = divmod(grp[ci[e]], gsz[1])
            got[(orb[ci[e]], ((h0 - t0) % gsz[0]) * gsz[1] + (h1 - t1) % gsz[1])] = va[e]
        assert got == rep[orb[r]]
