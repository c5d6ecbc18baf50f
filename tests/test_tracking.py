"""The reference's per-iteration bookkeeping on the fp32 hot path (run_pgd, solver.cpp:118-150):
E(x_0), E(x_k), support sizes, NonFiniteEnergy and the ref_energy stopping rule, computed by
the window engine's tracked kernel (fista_win_track_kernel: Theta x_k by linearity from the
next iteration's Theta y_k, no third SpMV). This is the path the drop-in binding's fista()
takes (integration/wbx_backend.cpp always asks for energies).

Bars: tracking leaves the iterates unchanged (x_final bitwise equal to the untracked fp32
solve); energies within 1e-5 relative of the reference's fp64 energies (fp32 iterates and
operator values); supports within 0.5 % of the reference's; the ref_energy rule stops at the
oracle's iteration wherever the oracle's energy is not within fp32 noise of the threshold."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_08401_b200 import synthetic as S
from paper_1512_08401_b200 import waveblur as W

pytestmark = pytest.mark.gpu

CASES = ["c1_db4_256", "s64_sym6_ista", "s32_sym4_naive", "s64_sym6_spai", "s128_1d_sym6"]


def setup(g):
    op = g.operator()
    b = W.make_basis(W.FilterFamily(g.family), g.meta["order"], g.dims, g.meta["J"])
    x0 = W.analyze(g["u0"].reshape(g.dims), b).values
    prob = W.DeblurProblem(W.SparseThetaOp(op), x0, g.weights(), g.meta["lambda"])
    kind = g.meta["precond"]
    if kind == "spai":
        P = W.spai(op)
    elif kind == "jacobi":
        gd = W.gram_diagonals(op)
        P = W.jacobi(op, max(1e-3 * gd.diagM.max(), 1e-300))
    else:
        P = W.identity_precond(op.n)
    return op, prob, P


@pytest.mark.parametrize("name", CASES)
def test_tracked_fp32_energies_and_iterates(golden, name, monkeypatch):
    monkeypatch.setenv("WBX_ENGINE", "window")  # untracked counterpart of the tracked window kernel
    g = golden(name)
    op, prob, P = setup(g)
    solve = W.ista if g.meta["method"] == "ista" else W.fista
    iters = g.meta["iters"]
    plain = solve(prob, P, W.SolverConfig(max_iters=iters, precision=32, track_energy=False))
    tr = solve(prob, P, W.SolverConfig(max_iters=iters, precision=32, track_energy=True, track_support=True))
    assert tr.iters_used == iters
    assert np.array_equal(tr.x_final, plain.x_final)  # bookkeeping does not touch the trajectory
    e, ref = np.array(tr.energies), np.asarray(g["energies"])
    assert e.shape == ref.shape
    assert np.max(np.abs(e - ref) / np.abs(ref)) < 1e-5
    assert abs(tr.initial_energy - g.meta["initial_energy"]) < 1e-5 * g.meta["initial_energy"]
    # supports against the fp64 reference mode (bitwise the reference's iterates)
    r64 = solve(prob, P, W.SolverConfig(max_iters=iters, precision=64, tau=g.meta["tau"], track_energy=True,
                                        track_support=True))
    s32, s64 = np.array(tr.support_sizes, dtype=np.int64), np.array(r64.support_sizes, dtype=np.int64)
    assert s32.shape == s64.shape
    assert np.all(np.abs(s32 - s64) <= np.maximum(2, 0.005 * s64))


@pytest.mark.parametrize("engine,kernel,tol", [(None, "circ_fista_kernel", 1e-9), ("window", "fista_win_track_kernel", 1e-5)])
def test_tracked_fp32_c2_1024_drop_in_path(golden, monkeypatch, engine, kernel, tol):
    """The 1024^2 headline operator through fista() with energies (the drop-in binding's call):
    the spectral engine (fp64; the reference's u0 is reproduced to 1e-12) and the tracked window
    kernel (fp32), energies against the reference's."""
    if engine:
        monkeypatch.setenv("WBX_ENGINE", engine)
    g = golden("c2_db4_1024")
    op = g.operator()
    b = W.make_basis(W.FilterFamily.Daubechies, 4, (1024, 1024), 4)
    _, u0 = S.degrade((1024, 1024), 5.0, 5e-3, 2024)  # the reference's u0 within 1e-12 (numpy FFT)
    x0 = W.analyze(u0, b).values
    prob = W.DeblurProblem(W.SparseThetaOp(op), x0, g.weights(), 1e-4)
    P = W.spai(op)
    d = W.Deblurrer(op, b, P, g.weights(), 1e-4, W.SolverConfig(max_iters=100, track_energy=True))
    assert d.kernels()[1] == kernel
    tr = W.fista(prob, P, W.SolverConfig(max_iters=100, precision=32, track_energy=True))
    e, ref = np.array(tr.energies), np.asarray(g["energies"])
    assert tr.iters_used == 100 and e.shape == ref.shape
    assert np.max(np.abs(e - ref) / np.abs(ref)) < tol, np.max(np.abs(e - ref) / np.abs(ref))


def test_tracked_fp32_ref_energy_rule_vs_oracle(golden):
    # solver.cpp:150, test_solver.cpp:263-289: stop once E(x_k) - E* <= tol * E(x_0)
    g = golden("s64_sym6_spai")
    op, prob, P = setup(g)
    estar = float(np.min(g["energies"]))
    A = O.Csr.of(op)
    AT = A.transpose()
    for accel, solve in ((True, W.fista), (False, W.ista)):
        cfg = W.SolverConfig(max_iters=2000, ref_energy=estar, precision=32)
        r = solve(prob, P, cfg)
        o = O.pgd(A, AT, prob.x0, prob.weights, prob.lambda_, P.p, 2000, accelerate=accel, ref_energy=estar,
                  energies=True)
        oe = np.asarray(o["energies"])
        gap = cfg.rel_energy_tol * o["initial_energy"]
        margin = np.abs(oe - estar - gap) / np.abs(oe)
        if np.all(margin[max(0, o["iters_used"] - 3):o["iters_used"]] > 1e-5):
            assert r.iters_used == o["iters_used"], (accel, r.iters_used, o["iters_used"])
        else:
            assert abs(r.iters_used - o["iters_used"]) <= 1
        assert len(r.energies) == r.iters_used
        assert r.energies[-1] - estar <= gap * (1 + 1e-6)


def test_tracked_fp32_nonfinite_energy(golden):
    g = golden("s32_sym4_naive")
    op, prob, _ = setup(g)
    I = W.identity_precond(op.n)
    with pytest.raises(W.NonFiniteEnergy):
        W.fista(prob, I, W.SolverConfig(max_iters=2000, precision=32, tau=1e6, track_energy=True))


def test_tracked_window_equals_stream_engine(golden, monkeypatch):
    """Window-engine tracking vs the streamed engine's (which spends the reference's third
    SpMV on E(x_k)): same iterates within fp32 noise, energies within 1e-6."""
    monkeypatch.setenv("WBX_ENGINE", "window")  # the fp32 window engine (not the spectral default)
    g = golden("c1_db4_256")
    op, prob, P = setup(g)
    cfg = W.SolverConfig(max_iters=50, precision=32, track_energy=True, track_support=True)
    a = W.fista(prob, P, cfg)
    monkeypatch.setenv("WBX_TRACK_ENGINE", "stream")
    b = W.fista(prob, P, cfg)
    ea, eb = np.array(a.energies), np.array(b.energies)
    assert np.max(np.abs(ea - eb) / np.abs(eb)) < 1e-6
    assert np.linalg.norm(a.x_final - b.x_final) <= 1e-5 * np.linalg.norm(b.x_final)
