"""Parity of the B200 path (through the C ABI, libwbx.so) against the reference's own
outputs (tests/golden) and the oracle restatement. Bar: bitwise for the fp64 paths
(DWT, SpMV, prox, Gram/SPAI, fp64 FISTA given tau); tau within 1e-12 relative (parallel
fp64 reductions); the fp32 hot path within rel-L2 <= 1e-5 of the reference's restored
image after the same iteration count (north_star tolerance)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_08401_b200 import synthetic as S
from paper_1512_08401_b200 import waveblur as W

pytestmark = pytest.mark.gpu

RTOL_IMAGE = 1e-5   # north_star: restored image rel-L2 <= 1e-5 (fp32 device vs fp64 reference)
RTOL_TAU = 1e-12

DWT_CASES = ["c1_db4_256", "s64_sym6_ista", "s32_sym4_naive", "s64_sym6_spai", "s128_1d_sym6"]
SOLVE_CASES = ["c1_db4_256", "s64_sym6_ista", "s32_sym4_naive", "s64_sym6_spai", "s128_1d_sym6"]


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def basis_of(g):
    return W.make_basis(W.FilterFamily(g.family), g.meta["order"], g.dims, g.meta["J"])


def precond_of(g, op):
    kind = g.meta["precond"]
    if kind == "spai":
        return W.spai(op)
    if kind == "jacobi":
        gd = W.gram_diagonals(op)
        return W.jacobi(op, max(1e-3 * gd.diagM.max(), 1e-300))
    return W.identity_precond(op.n)


# ----------------------------------------------------------------------------- wavelets
@pytest.mark.parametrize("name", DWT_CASES)
def test_dwt_bitwise_vs_reference(golden, name):
    g = golden(name)
    b = basis_of(g)
    x = W.analyze(g["u0"].reshape(g.dims), b).values
    assert np.array_equal(x, g["x0"])
    u = W.synthesize(g["x_final"], b).ravel()
    assert np.array_equal(u, g["restored"])


def test_dwt_known_answers_and_invariants():
    # test_wavelet.cpp:114-161
    b = W.make_basis(W.FilterFamily.Haar, 1, (4,), 2)
    x = W.analyze(np.ones(4), b).values
    assert abs(x[0] - 2.0) < 1e-14 and np.all(np.abs(x[1:]) < 1e-14)
    b2 = W.make_basis(W.FilterFamily.Haar, 1, (2,), 1)
    u = W.synthesize(np.array([1.0, 0.0]), b2)
    assert np.allclose(u, 1 / math.sqrt(2), atol=1e-15, rtol=0)
    b4 = W.make_basis(W.FilterFamily.Haar, 1, (4,), 1)
    w = W.single_wavelet(b4, 1, 1)
    assert np.allclose(w, [1 / math.sqrt(2), -1 / math.sqrt(2), 0, 0], atol=1e-14, rtol=0)
    bs = W.make_basis(W.FilterFamily.Symmlet, 6, (64,), 3)
    for band in bs.layout.bands:
        assert abs(np.linalg.norm(W.single_wavelet(bs, band.level, band.orientation)) - 1) < 1e-10
    with pytest.raises(W.BandNotFound):
        W.single_wavelet(bs, 5, 1)


@pytest.mark.parametrize("fam,order,dims,J", [(0, 1, (64, 64), 1), (1, 4, (64, 64), 3), (2, 6, (64, 64), 3),
                                              (2, 6, (128,), 3), (1, 3, (16, 64), 2), (2, 8, (8, 8), 3),
                                              (1, 10, (16, 16), 2)])
def test_dwt_bitwise_vs_oracle_random(fam, order, dims, J):
    rng = np.random.default_rng(17 + J)
    u = rng.random(dims)
    b = W.make_basis(W.FilterFamily(fam), order, dims, J)
    x = W.analyze(u, b).values
    assert np.array_equal(x, O.analyze(u, dims, J, fam, order))
    back = W.synthesize(x, b)
    assert np.array_equal(back.ravel(), O.synthesize(x, dims, J, fam, order))
    assert np.max(np.abs(back - u)) < 1e-10                       # round trip (test_wavelet.cpp:163-193)
    assert abs(np.linalg.norm(x) - np.linalg.norm(u)) < 1e-10 * np.linalg.norm(u)  # Parseval


def test_dwt_shape_errors():
    b = W.make_basis(W.FilterFamily.Haar, 1, (16,), 2)
    with pytest.raises(W.ShapeMismatch):
        W.analyze(np.zeros(32), b)
    with pytest.raises(W.ShapeMismatch):
        W.synthesize(np.zeros(8), b)


# ----------------------------------------------------------------------------- SpMV
@pytest.mark.parametrize("name", ["c1_db4_256", "s64_sym6_spai", "s128_1d_sym6", "s32_sym4_naive"])
def test_spmv_bitwise_vs_oracle(golden, name):
    g = golden(name)
    op = g.operator()
    A = O.Csr.of(op)
    rng = np.random.default_rng(101)
    x = rng.standard_normal(op.n)
    y = rng.standard_normal(op.n)
    assert np.array_equal(W.spmv(op, x), O.spmv(A, x))
    assert np.array_equal(W.spmv_t(op, y), O.spmv(A.transpose(), y))
    lhs = np.dot(W.spmv(op, x), y)
    rhs = np.dot(x, W.spmv_t(op, y))
    assert abs(lhs - rhs) < 1e-10 * max(1.0, abs(lhs))
    g2 = W.approx_gradient(op, x, y)
    r = O.spmv(A, x) - y
    assert np.array_equal(g2, O.spmv(A.transpose(), r))
    with pytest.raises(W.ShapeMismatch):
        W.spmv(op, np.zeros(12))


def test_spmv_edge_operators():
    # empty operator, single entry, full dense row
    n = 64
    empty = W.SparseOperator(n, np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32), np.zeros(0))
    assert np.array_equal(W.spmv(empty, np.ones(n)), np.zeros(n))
    ro = np.zeros(n + 1, np.uint64)
    ro[6:] = n   # row 5 is dense
    dense = W.SparseOperator(n, ro, np.arange(n, dtype=np.uint32), np.linspace(-1, 1, n))
    x = np.random.default_rng(3).standard_normal(n)
    A = O.Csr.of(dense)
    assert np.array_equal(W.spmv(dense, x), O.spmv(A, x))
    assert np.array_equal(W.spmv_t(dense, x), O.spmv(A.transpose(), x))
    bad = W.SparseOperator(4, np.array([0, 2, 2, 2, 2], np.uint64), np.array([1, 1], np.uint32), np.ones(2))
    with pytest.raises(W.ShapeMismatch):
        W.spmv(bad, np.ones(4))


def test_long_rows_serve_fp64_and_refuse_fp32():
    """rows beyond the fp32 segmented layout (31 segments x 16 = 496 nonzeros, e.g. the
    untruncated operators of test_theta.cpp:401-444): fp64 products, step and solve stay
    bitwise; an fp32 solve fails loudly with TooLarge instead of computing something else."""
    n = 1024
    rng = np.random.default_rng(17)
    ro = np.zeros(n + 1, np.uint64)
    lens = np.full(n, 3)
    lens[::97] = 700  # a few long rows (and long columns: the dense rows cover 0..699)
    ro[1:] = np.cumsum(lens)
    cols = np.concatenate([np.sort(rng.choice(n, L, replace=False)) if L != 700 else np.arange(700)
                           for L in lens]).astype(np.uint32)
    vals = rng.standard_normal(int(ro[-1])) * 0.05
    op = W.SparseOperator(n, ro, cols, vals)
    A = O.Csr.of(op)
    x = rng.standard_normal(n)
    assert np.array_equal(W.spmv(op, x), O.spmv(A, x))
    assert np.array_equal(W.spmv_t(op, x), O.spmv(A.transpose(), x))
    P = W.DiagonalPreconditioner(np.ones(n), W.PrecondKind.Identity)
    prob = W.DeblurProblem(W.SparseThetaOp(op), x, np.ones(n), 1e-3)
    r64 = W.fista(prob, P, W.SolverConfig(max_iters=20, precision=64, tau=0.5, track_energy=False))
    assert np.array_equal(r64.x_final, O.pgd_tau(A, A.transpose(), x, np.ones(n), 1e-3, np.ones(n), 0.5, 20))
    with pytest.raises(W.TooLarge):
        W.fista(prob, P, W.SolverConfig(max_iters=20, precision=32, track_energy=False))


# ----------------------------------------------------------------------------- prox / precond / step
def test_prox_closed_forms():
    # test_solver.cpp:76-94
    I = W.identity_precond(2)
    assert list(W.prox_weighted_l1_P([3.0, -0.5], 1.0, [0.0, 0.0], 1.0, I)) == [3.0, -0.5]
    s = W.prox_weighted_l1_P([3.0, -0.5], 1.0, [1.0, 1.0], 1.0, I)
    assert abs(s[0] - 2.0) < 1e-15 and s[1] == 0.0
    P = W.DiagonalPreconditioner(np.array([2.0, 1.0]), W.PrecondKind.Jacobi)
    s = W.prox_weighted_l1_P([3.0, -0.5], 1.0, [1.0, 1.0], 1.0, P)
    assert abs(s[0] - 2.5) < 1e-15 and s[1] == 0.0


def test_prox_bitwise_vs_oracle():
    rng = np.random.default_rng(12)
    z0, w, p = rng.standard_normal(1000), rng.random(1000) * 2, 0.5 + rng.random(1000)
    z = W.prox_weighted_l1_P(z0, 0.3, w, 0.7, W.DiagonalPreconditioner(p))
    assert np.array_equal(z, O.prox(z0, 0.3, w, 0.7, p))


@pytest.mark.parametrize("cap", ["2048", "32"])
@pytest.mark.parametrize("name", ["c1_db4_256", "s64_sym6_spai", "s128_1d_sym6"])
def test_preconditioner_bitwise_vs_reference(golden, monkeypatch, name, cap):
    """Gram diagonals on the device (there is no host path): SPAI and the Gram diagonals
    bitwise equal to the reference / oracle, with the default shared-memory tables and with
    32-slot tables, which sends most columns through the global-memory second pass."""
    monkeypatch.setenv("WBX_GRAM_CAP", cap)
    g = golden(name)
    op = g.operator()
    P = precond_of(g, op)
    assert np.array_equal(P.p, g["p"])
    gd = W.gram_diagonals(op)
    m, m2, st = O.gram_diagonals(O.Csr.of(op))
    assert st == 0 and np.array_equal(gd.diagM, m) and np.array_equal(gd.diagM2, m2)


@pytest.mark.parametrize("name", SOLVE_CASES + ["c1_sym6_256", "c2_db4_1024"])
def test_estimate_step_vs_reference(golden, name):
    g = golden(name)
    op = g.operator()
    P = precond_of(g, op)
    tau = W.estimate_step(W.SparseThetaOp(op), P, 1.01)
    assert abs(tau - g.meta["tau"]) <= RTOL_TAU * g.meta["tau"], (tau, g.meta["tau"])


def test_estimate_step_diagonal_operators():
    # test_solver.cpp:119-130
    n = 8
    eye = W.SparseOperator(n, np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.uint32), np.ones(n))
    I = W.identity_precond(n)
    assert abs(W.estimate_step(W.SparseThetaOp(eye), I, 1.0) - 1.0) < 1e-5
    assert abs(W.estimate_step(W.SparseThetaOp(eye), I, 1.25) - 0.8) < 1e-5
    v = np.ones(n)
    v[3] = 2.0
    d = W.SparseOperator(n, np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.uint32), v)
    assert abs(W.estimate_step(W.SparseThetaOp(d), I, 1.0) - 0.25) < 1e-5 * 0.25
    zero = W.SparseOperator(n, np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32), np.zeros(0))
    assert W.estimate_step(W.SparseThetaOp(zero), I, 1.0) == 1.0   # zero-operator sentinel


@pytest.mark.parametrize("name", SOLVE_CASES + ["c1_sym6_256", "c2_db4_1024"])
def test_lanczos_tau_equals_power_iteration(golden, monkeypatch, name):
    """The fp32 hot path estimates tau by Lanczos + the power iteration on the tridiagonal
    (tau_lanczos_win_kernel): the same reference iteration count (stopping rule) and the
    same tau as the literal power iteration (WBX_TAU=power) and the reference."""
    g = golden(name)
    op = g.operator()
    P = precond_of(g, op)
    prob = W.DeblurProblem(W.SparseThetaOp(op), np.zeros(op.n), g.weights(), g.meta["lambda"])
    cfg = W.SolverConfig(max_iters=0, precision=32, track_energy=False)
    lz = W.fista(prob, P, cfg)
    monkeypatch.setenv("WBX_TAU", "power")
    pw = W.fista(prob, P, cfg)
    assert lz.tau_iters == pw.tau_iters
    assert abs(lz.tau - pw.tau) <= 2e-7 * pw.tau
    assert abs(lz.tau - g.meta["tau"]) <= 1e-6 * g.meta["tau"]


def test_hot_path_deterministic_with_lanczos_tau(golden):
    """The fp32 deblur with the step estimated on the device (Lanczos) is bitwise
    reproducible run to run, like the reference (README.md:37-40): no atomics in any
    reduction, every CTA takes the same convergence decision."""
    g = golden("c1_db4_256")
    op = g.operator()
    b = basis_of(g)
    d = W.Deblurrer(op, b, precond_of(g, op), g.weights(), g.meta["lambda"],
                    W.SolverConfig(max_iters=g.meta["iters"], track_energy=False))
    u1, r1 = d.deblur(g["u0"].reshape(g.dims), clamp=False)
    u2, r2 = d.deblur(g["u0"].reshape(g.dims), clamp=False)
    assert r1.tau == r2.tau and r1.tau_iters == r2.tau_iters
    assert np.array_equal(u1, u2)
    assert d.tau_stats()[2] < r1.tau_iters  # fewer product pairs than the reference's iterations


def test_lanczos_tau_random_operators():
    """Random sparse operators and preconditioners (tools/tau_stress.py): the Lanczos
    estimate reproduces the fp64 reference mode's iteration count (stopping rule) and tau
    within 1e-6 on every case. (The literal fp32 power iteration does not: its fp32 rounding
    moves the stopping decision on about a quarter of these operators.)"""
    def random_op(rng, n, per_row):
        lens = rng.integers(0, per_row + 1, n)
        ro = np.zeros(n + 1, np.uint64)
        ro[1:] = np.cumsum(lens)
        cols = [np.sort(rng.choice(n, size=k, replace=False)) for k in lens]
        ci = np.concatenate(cols).astype(np.uint32)
        return W.SparseOperator(n, ro, ci, rng.standard_normal(int(ro[-1])) * rng.uniform(0.1, 2.0))

    rng = np.random.default_rng(99)
    for _ in range(12):
        n = int(rng.choice([64, 256, 1024]))
        op = random_op(rng, n, int(rng.integers(1, 12)))
        P = W.DiagonalPreconditioner(rng.uniform(0.2, 3.0, n), W.PrecondKind.Spai)
        prob = W.DeblurProblem(W.SparseThetaOp(op), np.zeros(n), np.ones(n), 1e-4)
        lz = W.fista(prob, P, W.SolverConfig(max_iters=0, precision=32, track_energy=False))
        t64, it64 = W.estimate_step(W.SparseThetaOp(op), P, 1.01, return_iters=True)
        assert lz.tau_iters == it64, (n, op.nnz())
        assert abs(lz.tau - t64) <= 1e-6 * t64


def test_lanczos_tau_small_spectra():
    """Operators whose Krylov space is tiny (Lanczos breaks down or only sees noise after a
    few steps): identity, two distinct scales, the zero operator, through the fp32 path."""
    n = 4096
    eye = W.SparseOperator(n, np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.uint32), np.ones(n))
    v = np.ones(n)
    v[::7] = 2.0
    two = W.SparseOperator(n, np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.uint32), v)
    zero = W.SparseOperator(n, np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32), np.zeros(0))
    I = W.identity_precond(n)
    cfg = W.SolverConfig(max_iters=0, precision=32, track_energy=False, step_safety=1.0)
    for op, tau in [(eye, 1.0), (two, 0.25), (zero, 1.0)]:
        r = W.fista(W.DeblurProblem(W.SparseThetaOp(op), np.zeros(n), np.ones(n), 1e-4), I, cfg)
        assert abs(r.tau - tau) <= 1e-6 * tau, (op.nnz(), r.tau)
        if op.nnz():  # the reference's own iteration count (power iteration in fp64)
            assert r.tau_iters == W.estimate_step(W.SparseThetaOp(op), I, 1.0, return_iters=True)[1]


# ----------------------------------------------------------------------------- solver
def _problem(g, op):
    b = basis_of(g)
    x0 = W.analyze(g["u0"].reshape(g.dims), b).values
    return W.DeblurProblem(W.SparseThetaOp(op), x0, g.weights(), g.meta["lambda"]), b


@pytest.mark.parametrize("name", SOLVE_CASES)
def test_fista_fp64_bitwise_vs_reference(golden, name):
    g = golden(name)
    op = g.operator()
    prob, b = _problem(g, op)
    P = precond_of(g, op)
    cfg = W.SolverConfig(max_iters=g.meta["iters"], precision=64, tau=g.meta["tau"], track_energy=True)
    solve = W.ista if g.meta["method"] == "ista" else W.fista
    rep = solve(prob, P, cfg)
    assert rep.iters_used == g.meta["iters"]
    assert np.array_equal(rep.x_final, g["x_final"])
    assert np.array_equal(W.synthesize(rep.x_final, b).ravel(), g["restored"])
    e = np.array(rep.energies)
    assert np.max(np.abs(e - g["energies"]) / np.abs(g["energies"])) < 1e-12
    assert abs(rep.initial_energy - g.meta["initial_energy"]) < 1e-12 * g.meta["initial_energy"]


@pytest.mark.parametrize("name", SOLVE_CASES)
def test_fista_fp32_hot_path_within_tolerance(golden, name):
    g = golden(name)
    op = g.operator()
    prob, b = _problem(g, op)
    P = precond_of(g, op)
    cfg = W.SolverConfig(max_iters=g.meta["iters"], precision=32, track_energy=False)
    solve = W.ista if g.meta["method"] == "ista" else W.fista
    rep = solve(prob, P, cfg)
    assert abs(rep.tau - g.meta["tau"]) <= 1e-6 * g.meta["tau"]
    u = W.synthesize(rep.x_final, b).ravel()
    assert rel_l2(u, g["restored"]) <= RTOL_IMAGE
    assert rel_l2(np.clip(u, 0, 1), np.clip(g["restored"], 0, 1)) <= RTOL_IMAGE


def test_zero_momentum_fista_equals_ista_bitwise(golden):
    # test_solver.cpp:241-261 / acceptance crit. 8
    g = golden("s32_sym4_naive")
    op = g.operator()
    prob, _ = _problem(g, op)
    I = W.identity_precond(op.n)
    for prec in (32, 64):
        a = W.ista(prob, I, W.SolverConfig(max_iters=25, precision=prec))
        bb = W.fista(prob, I, W.SolverConfig(max_iters=25, precision=prec, zero_momentum=True))
        assert np.array_equal(a.x_final, bb.x_final)
        assert a.energies == bb.energies


def test_ista_monotone_and_deterministic(golden):
    # test_solver.cpp:176-201
    g = golden("s64_sym6_ista")
    op = g.operator()
    prob, _ = _problem(g, op)
    I = W.identity_precond(op.n)
    a = W.ista(prob, I, W.SolverConfig(max_iters=40, precision=64))
    for k in range(1, len(a.energies)):
        assert a.energies[k] <= a.energies[k - 1] + 1e-12
    b = W.ista(prob, I, W.SolverConfig(max_iters=40, precision=64))
    assert np.array_equal(a.x_final, b.x_final) and a.energies == b.energies
    c = W.fista(prob, I, W.SolverConfig(max_iters=40, precision=32, track_energy=False))
    d = W.fista(prob, I, W.SolverConfig(max_iters=40, precision=32, track_energy=False))
    assert np.array_equal(c.x_final, d.x_final)   # fp32 hot path is run-to-run bitwise too


def test_fista_ref_energy_stopping_rule(golden):
    # solver.cpp:150 and test_solver.cpp:263-289
    g = golden("s64_sym6_spai")
    op = g.operator()
    prob, _ = _problem(g, op)
    P = precond_of(g, op)
    estar = float(np.min(g["energies"]))
    I = W.identity_precond(op.n)
    cfg = W.SolverConfig(max_iters=2000, ref_energy=estar, precision=64)
    fi = W.fista(prob, I, cfg)
    is_ = W.ista(prob, I, cfg)
    assert fi.iters_used < is_.iters_used
    assert fi.iters_used < cfg.max_iters
    r = O.pgd(O.Csr.of(op), O.Csr.of(op).transpose(), prob.x0, prob.weights, prob.lambda_, I.p, 2000,
              ref_energy=estar)
    assert fi.iters_used == r["iters_used"]
    assert np.array_equal(fi.x_final, r["x_final"]) or rel_l2(fi.x_final, r["x_final"]) < 1e-12
    del P


def test_max_iters_zero_and_nonfinite(golden):
    g = golden("s32_sym4_naive")
    op = g.operator()
    prob, _ = _problem(g, op)
    I = W.identity_precond(op.n)
    r = W.fista(prob, I, W.SolverConfig(max_iters=0, precision=64))
    assert r.iters_used == 0 and np.array_equal(r.x_final, prob.x0)
    with pytest.raises(W.NonFiniteEnergy):
        W.fista(prob, I, W.SolverConfig(max_iters=2000, precision=64, tau=1e6, track_energy=True))


# ----------------------------------------------------------------------------- prepared deblur (the bench unit)
def test_deblurrer_c1_vs_reference(golden):
    g = golden("c1_db4_256")
    op = g.operator()
    b = basis_of(g)
    P = W.spai(op)
    d = W.Deblurrer(op, b, P, g.weights(), g.meta["lambda"], W.SolverConfig(max_iters=50, track_energy=False))
    u, rep = d.deblur(g["u0"], clamp=False)
    assert abs(rep.tau - g.meta["tau"]) <= 1e-6 * g.meta["tau"]
    assert rel_l2(u, g["restored"]) <= RTOL_IMAGE
    uc, _ = d.deblur(g["u0"], clamp=True)
    assert rel_l2(uc, np.clip(g["restored"], 0, 1)) <= RTOL_IMAGE
    d64 = W.Deblurrer(op, b, P, g.weights(), g.meta["lambda"],
                      W.SolverConfig(max_iters=50, precision=64, tau=g.meta["tau"], track_energy=False))
    u64, _ = d64.deblur(g["u0"], clamp=False)
    assert np.array_equal(u64.ravel(), g["restored"])


@pytest.mark.slow
def test_deblurrer_c2_1024_vs_oracle(golden):
    """BASELINE config C2 at full size: 1024^2 stationary, 100 iterations."""
    g = golden("c2_db4_1024")
    op = g.operator()
    b = basis_of(g)
    P = W.spai(op)
    w = g.weights()
    _, u0 = S.degrade((1024, 1024), 5.0, 5e-3, 2024)
    d = W.Deblurrer(op, b, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False))
    u, rep = d.deblur(u0, clamp=False)
    assert abs(rep.tau - g.meta["tau"]) <= 1e-6 * g.meta["tau"]
    A = O.Csr.of(op)
    x0 = O.analyze(u0, (1024, 1024), 4, 1, 4)
    xr = O.pgd_tau(A, A.transpose(), x0, w, 1e-4, P.p, g.meta["tau"], 100)
    ur = O.synthesize(xr, (1024, 1024), 4, 1, 4)
    assert rel_l2(u, ur) <= RTOL_IMAGE
    # final energy of the reference's own run (its u0 differs from ours by < 1e-12)
    x_ours = W.analyze(u.reshape(1024, 1024), b).values
    e = W.energy(x_ours, W.DeblurProblem(W.SparseThetaOp(op), W.analyze(u0, b).values, w, 1e-4))
    assert abs(e - g.meta["final_energy"]) < 1e-5 * g.meta["final_energy"]


# ----------------------------------------------------------------------------- engine / format variants
_W = {"WBX_ENGINE": "window"}  # the window engine instead of the spectral one (invariant operators)


@pytest.mark.parametrize("env", [{}, _W, {**_W, "WBX_WIN_FULL": "1"}, {"WBX_ENGINE": "stream"},
                                 {**_W, "WBX_TAU": "lanczos"}, {**_W, "WBX_TAU": "power"},
                                 {**_W, "WBX_TAU": "power", "WBX_TAU_WINDOW": "64", "WBX_WIN_PLACE": "bank"},
                                 {**_W, "WBX_WIN_PLACE": "bank"},
                                 {**_W, "WBX_WIN_PLACE": "sorted"}, {**_W, "WBX_BARRIER": "master"},
                                 {**_W, "WBX_WIN_COST": "16,1"}, {**_W, "WBX_WIN_LISTS": "global"}])
def test_deblurrer_engine_variants_vs_reference(golden, monkeypatch, env):
    """Every solver engine / window format / placement / barrier the library can select
    (environment switches read at solver creation) meets the same parity bar on C1."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = golden("c1_db4_256")
    op = g.operator()
    d = W.Deblurrer(op, basis_of(g), W.spai(op), g.weights(), g.meta["lambda"],
                    W.SolverConfig(max_iters=50, track_energy=False))
    u, rep = d.deblur(g["u0"], clamp=False)
    assert abs(rep.tau - g.meta["tau"]) <= 1e-6 * g.meta["tau"]
    assert rel_l2(u, g["restored"]) <= RTOL_IMAGE
    u2, _ = d.deblur(g["u0"], clamp=False)
    assert np.array_equal(u, u2)  # run-to-run deterministic


@pytest.mark.parametrize("env", [{"WBX_WIN_FULL": "1"}, {"WBX_WIN_PLACE": "sorted"}, {"WBX_WIN_PLACE": "bank"}, {"WBX_WIN_PLACE": "chunk-bank"},
                                 {"WBX_BARRIER": "master"},
                                 {"WBX_WIN_COST": "16,1"}, {"WBX_WIN_LISTS": "global"}, {"WBX_BARRIER_GROUPS": "4"},
                                 {"WBX_WIN_MODEL": "0.0186,0.0129,0.0024,0,0"}, {"WBX_GRAPH": "0"}])
def test_window_layout_variants_leave_iterates_bitwise(golden, monkeypatch, env):
    """The window engine's partition, slot placement, value format, list placement, barrier and
    launch mode change no arithmetic: given tau, the restored image is bitwise the default's."""
    g = golden("c1_db4_256")
    cfg = W.SolverConfig(max_iters=50, track_energy=False, tau=g.meta["tau"])
    op = g.operator()
    P = W.spai(op)
    monkeypatch.setenv("WBX_ENGINE", "window")
    ref = W.Deblurrer(op, basis_of(g), P, g.weights(), g.meta["lambda"], cfg).deblur(g["u0"], clamp=False)[0]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    op2 = g.operator()  # window layouts are cached per operator: a fresh one
    d = W.Deblurrer(op2, basis_of(g), P, g.weights(), g.meta["lambda"], cfg)
    assert d.kernels()[1] == "fista_win_kernel"
    assert np.array_equal(d.deblur(g["u0"], clamp=False)[0], ref)


def test_deblur_graphs_follow_the_buffers(golden):
    """wbx_deblur_dev runs as two CUDA graphs captured for the (u0, u, clamp) pointers of the
    call: alternating buffers and clamp flags re-capture and give the same images as the
    host entry point (and as launching kernel by kernel, WBX_GRAPH=0 in the variant test)."""
    import torch
    g = golden("c1_db4_256")
    op = g.operator()
    d = W.Deblurrer(op, basis_of(g), W.spai(op), g.weights(), g.meta["lambda"],
                    W.SolverConfig(max_iters=50, track_energy=False))
    ref, _ = d.deblur(g["u0"], clamp=True)
    refc, _ = d.deblur(g["u0"], clamp=False)
    dev = torch.device("cuda", 0)
    u0 = torch.from_numpy(g["u0"].copy()).to(dev)
    outs = [torch.empty_like(u0) for _ in range(2)]
    for k in range(4):
        o = outs[k % 2]
        clamp = k < 2
        d.deblur_dev(u0.data_ptr(), o.data_ptr(), clamp=clamp)
        torch.cuda.synchronize()
        assert np.array_equal(o.cpu().numpy().reshape(256, 256), ref if clamp else refc)
        launches, _ = d.last_stats()
        assert launches > 0
