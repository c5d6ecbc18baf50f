"""BASELINE configs C3/C4: spatially varying blur. The reference has no 2-D spatially varying
operator, so Theta_K construction parity is unpinned; its ingredients are
the reference's own stationary operators (tests/golden/c3_ladder_*.npz) and the SOLVER
parity stays pinned: the oracle runs the same CSR."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_08401_b200 import synthetic as S
from paper_1512_08401_b200 import waveblur as W
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


def ladder(size):
    return W.SigmaLadder.from_npz(np.load(GOLDEN / f"c3_ladder_{size}.npz"))


def test_flat_sigma_reproduces_the_stationary_level():
    lad = ladder(256)
    for l in (0, 3, 7):
        s = lad.sigmas[l]
        op = W.theta_varying(lad, s, s)
        ref = W.theta_from_generators(lad.levels[l])
        assert np.array_equal(op.row_offsets, ref.row_offsets)
        assert np.array_equal(op.col_indices, ref.col_indices)
        assert np.array_equal(op.values, ref.values)


def test_varying_columns_interpolate_bracketing_levels():
    lad = ladder(256)
    op = W.theta_varying(lad, 2.5, 7.5)
    assert op.nnz() > 3 * op.n  # union of two levels' index sets per column
    ro = op.row_offsets.astype(np.int64)
    rows = np.repeat(np.arange(op.n), np.diff(ro))
    same = rows[1:] == rows[:-1]
    assert np.all(op.col_indices[1:][same] > op.col_indices[:-1][same])
    # a column at the top of the image is (nearly) the sigma=2.5 operator's column, at the
    # bottom the sigma=7.5 one: compare one coarse-band column each against the levels
    dense = lambda o, c: {int(r): v for r, v in zip(rows[o.col_indices == c], o.values[o.col_indices == c])}
    lv0 = W.theta_from_generators(lad.levels[0])
    r0 = np.repeat(np.arange(lv0.n), np.diff(lv0.row_offsets.astype(np.int64)))
    c = 0  # band 0, row 0: y = 8 px of 256 -> sigma = 2.656, between levels 0 and 1
    a = dense(op, c)
    b = {int(r): v for r, v in zip(r0[lv0.col_indices == c], lv0.values[lv0.col_indices == c])}
    common = set(a) & set(b)
    assert len(common) > 10
    rel = max(abs(a[k] - b[k]) / abs(b[k]) for k in common)
    assert rel < 0.5


def test_varying_rejects_bad_ladder():
    lad = ladder(256)
    bad = W.SigmaLadder(lad.sigmas[::-1].copy(), lad.levels[::-1])
    with pytest.raises(W.BadSpec):
        W.theta_varying(bad, 2.5, 7.5)


def varying_input(op, basis, seed=2024):
    """u0 = Psi Theta_var Psi^* u_clean + noise, with the oracle's exact fp64 transforms."""
    dims = basis.layout.dims
    clean = S.synthetic_scene(dims)
    fam, order, J = int(basis.filters.family), basis.filters.order, basis.layout.J
    x = O.analyze(clean, dims, J, fam, order)
    bx = O.spmv(O.Csr.of(op), x)
    u = O.synthesize(bx, dims, J, fam, order).reshape(dims)
    return clean, S.add_noise(u, 5e-3, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("size,iters", [(256, 50), (1024, 100)])
def test_c3_deblur_matches_oracle(size, iters):
    lad = ladder(size)
    op = W.theta_varying(lad, 2.5, 7.5)
    basis = W.make_basis(W.FilterFamily.Daubechies, 4, (size, size), 4)
    clean, u0 = varying_input(op, basis)
    P = W.spai(op)
    w = W.scale_weights(basis.layout)
    d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=iters, track_energy=False))
    u, rep = d.deblur(u0, clamp=False)
    A = O.Csr.of(op)
    AT = A.transpose()
    p_ref = O.spai(A)
    assert np.array_equal(P.p, p_ref)
    tau_ref, _ = O.estimate_step(A, AT, p_ref, 1.01)
    assert abs(rep.tau - tau_ref) <= 1e-6 * tau_ref
    x0 = O.analyze(u0, (size, size), 4, 1, 4)
    xr = O.pgd_tau(A, AT, x0, w, 1e-4, p_ref, tau_ref, iters)
    ur = O.synthesize(xr, (size, size), 4, 1, 4)
    err = np.linalg.norm(u.ravel() - ur) / np.linalg.norm(ur)
    assert err <= 1e-5, err
    assert S.psnr(np.clip(u, 0, 1), clean) > S.psnr(u0, clean)  # it deblurs


def test_rescaled_generators_reproduce_the_reference_at_1024():
    """C4 derives 4096^2 operators by rescaling; check the rule where the reference itself is
    available: the 256^2 lists rescaled to 1024^2 give the reference's 1024^2 operator (same
    index set; values equal to ~1e-13, the periodisation difference of the two grids)."""
    z256, z1024 = np.load(GOLDEN / "c1_db4_256.npz"), np.load(GOLDEN / "c2_db4_1024.npz")
    mk = lambda z, d: W.GeneratorList(d, 4, W.FilterFamily.Daubechies, 4, z["gen_block"].astype(np.uint32),
                                      z["gen_index"].astype(np.uint32), z["gen_count"].astype(np.uint64),
                                      z["gen_value"])
    a = W.theta_from_generators(W.rescale_generators(mk(z256, (256, 256)), (1024, 1024)))
    b = W.theta_from_generators(mk(z1024, (1024, 1024)))
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert np.max(np.abs(a.values - b.values) / np.abs(b.values)) < 1e-12
