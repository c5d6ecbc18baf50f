"""The stencil engine's FISTA kernel (fista_stencil_kernel, csrc/stencil_kernel.cuh): FISTA
iterations on a stationary Theta_K straight from its generator groups (no index stream).

Parity: the restored image after the reference's iteration count against the oracle's fp64
run_pgd restatement (oracle/wbx_oracle.c `pgd_tau`, pinned bitwise to the reference) on the
same CSR, preconditioner and tau: rel-L2 <= 1e-5 (north_star's bar); against the reference's
own restored image where the fixture holds it (C1); and against the window engine (same fp32
arithmetic, different summation order) within fp32 rounding."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_08401_b200 import synthetic as S
from paper_1512_08401_b200 import waveblur as W

pytestmark = pytest.mark.gpu

RTOL_IMAGE = 1e-5


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


def solve(g, monkeypatch, engine, u0, iters):
    if engine == "stencil":
        monkeypatch.setenv("WBX_STENCIL", "1")
    else:
        monkeypatch.delenv("WBX_STENCIL", raising=False)
        monkeypatch.setenv("WBX_ENGINE", engine)  # the fp32 window engine (not the spectral default)
    op = g.operator()
    basis = W.make_basis(W.FilterFamily(g.family), g.meta["order"], g.dims, g.meta["J"])
    P = W.spai(op)
    d = W.Deblurrer(op, basis, P, g.weights(), g.meta["lambda"], W.SolverConfig(max_iters=iters, track_energy=False))
    u, rep = d.deblur(u0, clamp=False)
    return op, basis, P, d, u, rep


@pytest.mark.parametrize("name", ["c1_db4_256", "c1_sym6_256", "c2_db4_1024"])
def test_stencil_engine_vs_oracle(golden, monkeypatch, name):
    g = golden(name)
    u0 = g["u0"] if "u0" in g else S.degrade(g.dims, 5.0, 5e-3, g.meta["seed"])[1].ravel()
    iters = g.meta["iters"]
    op, basis, P, d, u, rep = solve(g, monkeypatch, "stencil", u0, iters)
    assert "fista_stencil_kernel" in d.kernels()
    assert abs(rep.tau - g.meta["tau"]) <= 1e-6 * g.meta["tau"]
    if "restored" in g:
        assert rel_l2(u, g["restored"]) <= RTOL_IMAGE
    J, order, fam = g.meta["J"], g.meta["order"], g.family
    A = O.Csr.of(op)
    xr = O.pgd_tau(A, A.transpose(), O.analyze(np.asarray(u0, dtype=np.float64).reshape(g.dims), g.dims, J, fam, order),
                   g.weights(), g.meta["lambda"], P.p, rep.tau, iters)
    ur = O.synthesize(xr, g.dims, J, fam, order)
    assert rel_l2(u, ur) <= RTOL_IMAGE
    _, _, _, dw, uw, _ = solve(g, monkeypatch, "window", u0, iters)
    assert "fista_stencil_kernel" not in dw.kernels()
    assert rel_l2(u, uw) <= 2e-6


def test_stencil_engine_repeatable_and_clamped(golden, monkeypatch):
    g = golden("c1_db4_256")
    _, _, _, d, u, _ = solve(g, monkeypatch, "stencil", g["u0"], 50)
    u2, _ = d.deblur(g["u0"], clamp=False)
    assert np.array_equal(u, u2)
    uc, _ = d.deblur(g["u0"], clamp=True)
    assert np.array_equal(uc, np.clip(u, 0, 1))
