"""Spectral FISTA engine (csrc/circ_tau.cu circ_fista_kernel) through the C ABI.

For a translation-invariant Theta_K the solver applies the gradient Theta^T (Theta y - x0) as
G y - b with G block-diagonal in the Fourier domain of the translation group (G_f =
Theta^_f^H Theta^_f, 12 x 12 at C1/C2), in fp64, with the reference's prox / momentum /
threshold expressions (solver.cpp:57-67, 119-151). Bar: the iterates of the reference's fp64
run_pgd to ~1e-12 (vs 1e-5 for the fp32 window engine): restored images against the
reference's golden outputs and the oracle's pgd on the same inputs."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_08401_b200 import waveblur as W

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def setup(g):
    op = g.operator()
    b = W.make_basis(W.FilterFamily(g.family), g.meta["order"], g.dims, g.meta["J"])
    return op, b, W.spai(op)


def test_spectral_deblur_vs_reference(golden):
    g = golden("c1_db4_256")
    op, b, P = setup(g)
    d = W.Deblurrer(op, b, P, g.weights(), g.meta["lambda"], W.SolverConfig(max_iters=g.meta["iters"], track_energy=False))
    assert d.kernels() == ("circ_lanczos_kernel", "circ_fista_kernel")
    u, rep = d.deblur(g["u0"], clamp=False)
    err = rel_l2(u, g["restored"])
    print("C1 restored rel-L2 vs the reference:", err)
    assert err <= 1e-11
    x = W.analyze(u.reshape(g.dims), b).values
    assert rel_l2(x, g["x_final"]) <= 1e-10
    u2, _ = d.deblur(g["u0"], clamp=False)
    assert np.array_equal(u, u2)  # run-to-run deterministic


@pytest.mark.parametrize("iters", [0, 1, 2, 7])
def test_spectral_iterates_vs_oracle_given_tau(golden, iters):
    """Given tau (the gram blocks then come from the iteration launch): x_final vs the oracle's
    fp64 pgd (pinned bitwise to the reference) for short runs, including K = 0."""
    g = golden("c1_db4_256")
    op, b, P = setup(g)
    tau = g.meta["tau"]
    d = W.Deblurrer(op, b, P, g.weights(), g.meta["lambda"],
                    W.SolverConfig(max_iters=iters, track_energy=False, tau=tau))
    assert d.kernels()[1] == "circ_fista_kernel"
    u, _ = d.deblur(g["u0"], clamp=False)
    A = O.Csr.of(op)
    xr = O.pgd_tau(A, A.transpose(), g["x0"], g.weights(), g.meta["lambda"], P.p, tau, iters)
    ur = O.synthesize(xr, g.dims, g.meta["J"], g.family, g.meta["order"])
    assert rel_l2(u, ur) <= 1e-12, rel_l2(u, ur)


def test_spectral_sym6_and_ista_case(golden):
    """Another filter family and the ISTA-style identity-preconditioned invariant case."""
    g = golden("s64_sym6_ista")
    op, b, _ = setup(g)
    P = W.identity_precond(op.n)
    tau = g.meta["tau"]
    d = W.Deblurrer(op, b, P, g.weights(), g.meta["lambda"], W.SolverConfig(max_iters=20, track_energy=False, tau=tau))
    assert d.kernels()[1] == "circ_fista_kernel"
    u, _ = d.deblur(g["u0"], clamp=False)
    A = O.Csr.of(op)
    xr = O.pgd_tau(A, A.transpose(), g["x0"], g.weights(), g.meta["lambda"], P.p, tau, 20)
    ur = O.synthesize(xr, g.dims, g.meta["J"], g.family, g.meta["order"])
    assert rel_l2(u, ur) <= 1e-12, rel_l2(u, ur)


def test_tracked_and_window_engines_still_selected(golden, monkeypatch):
    """Tracked solves without the ref_energy rule run on the spectral engine; the ref_energy rule
    keeps the window engine; WBX_ENGINE=window forces it for the others."""
    g = golden("c1_db4_256")
    op, b, P = setup(g)
    d = W.Deblurrer(op, b, P, g.weights(), g.meta["lambda"], W.SolverConfig(max_iters=5, track_energy=True))
    assert d.kernels()[1] == "circ_fista_kernel"
    d = W.Deblurrer(op, b, P, g.weights(), g.meta["lambda"],
                    W.SolverConfig(max_iters=5, track_energy=True, ref_energy=1.0))
    assert d.kernels()[1] == "fista_win_track_kernel"
    monkeypatch.setenv("WBX_ENGINE", "window")
    d = W.Deblurrer(op, b, P, g.weights(), g.meta["lambda"], W.SolverConfig(max_iters=5, track_energy=False))
    assert d.kernels()[1] == "fista_win_kernel"


@pytest.mark.parametrize("name", ["c1_db4_256", "s64_sym6_ista"])
def test_tracked_spectral_energies_vs_reference(golden, name):
    """The reference's own fista() with its per-iteration energies and supports (the drop-in
    binding's call) on the spectral engine: energies, the initial energy and the supports of the
    reference's run, x_final as the untracked solve's."""
    g = golden(name)
    op, b, P = setup(g)
    if g.meta["precond"] == "identity":
        P = W.identity_precond(op.n)
    prob = W.DeblurProblem(W.SparseThetaOp(op), g["x0"], g.weights(), g.meta["lambda"])
    iters = g.meta["iters"]
    solve = W.ista if g.meta.get("method") == "ista" else W.fista
    tr = solve(prob, P, W.SolverConfig(max_iters=iters, precision=32, track_energy=True, track_support=True))
    plain = solve(prob, P, W.SolverConfig(max_iters=iters, precision=32, track_energy=False))
    assert tr.iters_used == iters
    assert np.array_equal(tr.x_final, plain.x_final)  # bookkeeping does not touch the trajectory
    e, ref = np.array(tr.energies), np.asarray(g["energies"])
    assert e.shape == ref.shape
    assert np.max(np.abs(e - ref) / np.abs(ref)) <= 1e-10, np.max(np.abs(e - ref) / np.abs(ref))
    assert abs(tr.initial_energy - g.meta["initial_energy"]) <= 1e-10 * abs(g.meta["initial_energy"])
    assert len(tr.support_sizes) == iters
    assert tr.support_sizes[-1] == int(np.count_nonzero(tr.x_final))  # support of the last iterate


@pytest.mark.parametrize("dims,fam,order,J", [((64, 64), W.FilterFamily.Haar, 1, 1),     # g = 32, 1 column orbit
                                              ((128, 128), W.FilterFamily.Daubechies, 2, 2),  # g = 32
                                              ((128, 128), W.FilterFamily.Symmlet, 4, 3)])    # g = 16
def test_spectral_other_groups_vs_oracle(dims, fam, order, J):
    """Operators built on the device (theta_conv_topk) whose column-orbit count is not a multiple
    of the engine's row padding, and other group sizes: the whole deblur vs the oracle's pgd."""
    from paper_1512_08401_b200 import synthetic as S
    basis = W.make_basis(fam, order, dims, J)
    n = basis.layout.total()
    op = W.theta_from_generators(W.theta_conv_topk(basis, W.gaussian_psf_kernel(dims, 2.5), 3 * n,
                                                   W.dyadic_band_weights(basis.layout)))
    P = W.spai(op)
    u0 = S.add_noise(W.synthesize(W.spmv(op, W.analyze(S.synthetic_scene(dims), basis).values), basis), 5e-3, 4)
    w = W.scale_weights(basis.layout)
    d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=30, track_energy=False))
    u, rep = d.deblur(u0, clamp=False)
    A = O.Csr.of(op)
    ref = O.pgd(A, A.transpose(), O.analyze(u0, dims, J, int(fam), order), w, 1e-4, P.p, 30)
    assert abs(rep.tau - ref["tau"]) <= 1e-12 * ref["tau"]
    if d.kernels()[1] == "circ_fista_kernel":
        ur = O.synthesize(ref["x_final"], dims, J, int(fam), order)
        assert rel_l2(u, ur) <= 1e-12, rel_l2(u, ur)


def test_dropin_fista_solver_cache_reuse(golden):
    """wbx_pgd keeps solvers across calls (same operator and configuration): new P, w, lambda
    and x0 are taken into account every call, and a repeated call gives the same bits."""
    g = golden("c1_db4_256")
    op = g.operator()
    P1 = W.spai(op)
    rng = np.random.default_rng(5)
    P2 = W.DiagonalPreconditioner(P1.p * rng.uniform(0.8, 1.25, op.n), W.PrecondKind.Spai)  # not orbit-constant
    A = O.Csr.of(op)
    cfg = W.SolverConfig(max_iters=20, precision=32, track_energy=False)
    w = g.weights()
    runs = []
    for P, lam, x0 in [(P1, 1e-4, g["x0"]), (P2, 3e-4, g["x0"]), (P1, 1e-4, 0.5 * g["x0"]), (P1, 1e-4, g["x0"])]:
        r = W.fista(W.DeblurProblem(W.SparseThetaOp(op), x0, w, lam), P, cfg)
        ref = O.pgd(A, A.transpose(), x0, w, lam, P.p, 20)
        assert abs(r.tau - ref["tau"]) <= 1e-6 * ref["tau"]
        assert rel_l2(r.x_final, ref["x_final"]) <= 1e-5
        runs.append(r.x_final)
    assert np.array_equal(runs[0], runs[3])


@pytest.mark.parametrize("batch,slots", [(4, None), (8, None), (8, "1"), (8, "3")])
def test_spectral_batch_bitwise_equals_single(golden, batch, slots, monkeypatch):
    """C5 on the spectral engine: a batch solves its images `slots` per launch (NB spectral CTAs,
    an exchange buffer and a barrier counter per image; the decoupled CTAs take every image's
    decoupled coordinates). Each image must equal its single-image spectral solve bitwise; the
    golden image inside the batch matches the reference's restored image."""
    if slots:
        monkeypatch.setenv("WBX_CIRC_SLOTS", slots)
    from paper_1512_08401_b200 import synthetic as S
    g = golden("c1_db4_256")
    op, b, P = setup(g)
    cfg = W.SolverConfig(max_iters=g.meta["iters"], track_energy=False)
    imgs = np.stack([g["u0"].reshape(g.dims)] +
                    [S.degrade(g.dims, 5.0, 5e-3, seed)[1] for seed in range(1, batch)])
    single = W.Deblurrer(op, b, P, g.weights(), g.meta["lambda"], cfg)
    ref = np.stack([single.deblur(im, clamp=False)[0] for im in imgs])
    many = W.Deblurrer(op, b, P, g.weights(), g.meta["lambda"], cfg, batch=batch)
    assert many.kernels() == ("circ_lanczos_kernel", "circ_fista_kernel")
    out, rep = many.deblur(imgs, clamp=False)
    assert out.shape == (batch,) + tuple(g.dims)
    assert np.array_equal(out, ref)
    assert rel_l2(out[0], g["restored"]) <= 1e-11
    assert abs(rep.tau - g.meta["tau"]) <= 1e-12 * g.meta["tau"]
    out2, _ = many.deblur(imgs, clamp=False)
    assert np.array_equal(out, out2)


@pytest.mark.parametrize("batch", [4, 8])
def test_spectral_batch_at_1024(golden, batch):
    """C5 at its real size: 4 / 8 images of the C2 operator in one launch (64 spectral CTAs per
    slot, 2 / 4 images per CTA: circ_fista_multi_kernel) bitwise equal to single-image spectral
    solves (whose parity with the reference is pinned above and in test_full_size), tau the
    reference's."""
    from paper_1512_08401_b200 import synthetic as S
    g = golden("c2_db4_1024")
    op = g.operator()
    ctx = W.Context(0)
    b = W.make_basis(W.FilterFamily.Daubechies, 4, (1024, 1024), 4)
    P = W.spai(op, ctx)
    cfg = W.SolverConfig(max_iters=100, track_energy=False)
    imgs = np.stack([S.degrade((1024, 1024), 5.0, 5e-3, seed)[1] for seed in range(batch)])
    single = W.Deblurrer(op, b, P, g.weights(), 1e-4, cfg, ctx)
    ref = np.stack([single.deblur(im, clamp=True)[0] for im in imgs])
    many = W.Deblurrer(op, b, P, g.weights(), 1e-4, cfg, ctx, batch=batch)
    assert many.kernels() == ("circ_lanczos_kernel", "circ_fista_kernel")
    out, rep = many.deblur(imgs, clamp=True)
    assert np.array_equal(out, ref)
    assert abs(rep.tau - g.meta["tau"]) <= 1e-12 * g.meta["tau"]


@pytest.mark.parametrize("multi", ["1", "0"])
def test_spectral_batch8_at_512_two_images_per_cta(multi, monkeypatch):
    """g = 32 (512^2, J = 4): 4 CTA slots of 32 spectral CTAs, so a batch of 8 runs 2 images per
    CTA in one launch (WBX_CIRC_MULTI=0: one image per CTA, two launches); Theta_K built on the
    device from the Gaussian PSF (sigma 5, K = 3N, dyadic weights). Bitwise equal to single-image solves."""
    if multi == "0":
        monkeypatch.setenv("WBX_CIRC_MULTI", "0")
    from paper_1512_08401_b200 import synthetic as S
    dims = (512, 512)
    ctx = W.Context(0)
    b = W.make_basis(W.FilterFamily.Daubechies, 4, dims, 4)
    n = dims[0] * dims[1]
    gl = W.theta_conv_topk(b, W.gaussian_psf_kernel(dims, 5.0), 3 * n, W.dyadic_band_weights(b.layout), ctx)
    op = W.theta_from_generators(gl)
    P = W.spai(op, ctx)
    w = W.scale_weights(b.layout)
    cfg = W.SolverConfig(max_iters=30, track_energy=False)
    imgs = np.stack([S.degrade(dims, 5.0, 5e-3, seed)[1] for seed in range(8)])
    single = W.Deblurrer(op, b, P, w, 1e-4, cfg, ctx)
    assert single.kernels() == ("circ_lanczos_kernel", "circ_fista_kernel")
    ref = np.stack([single.deblur(im, clamp=False)[0] for im in imgs])
    many = W.Deblurrer(op, b, P, w, 1e-4, cfg, ctx, batch=8)
    out, _ = many.deblur(imgs, clamp=False)
    assert np.array_equal(out, ref)
