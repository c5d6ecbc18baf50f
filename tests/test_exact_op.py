"""ExactThetaOp on the device: the exact FFT operator and the exact-fista
comparator, against the REFERENCE's own ExactThetaOp outputs (tests/golden/exact_s64_sym6,
written by oracle/tools/oracle_driver.cpp --exact)."""
import numpy as np
import pytest

from paper_1512_08401_b200 import waveblur as W

pytestmark = pytest.mark.gpu


def _setup(golden):
    g = golden("exact_s64_sym6")
    m = g.meta
    dims = tuple(m["dims"])
    basis = W.make_basis(W.FilterFamily(g.family), m["order"], dims, m["J"])
    return g, m, dims, basis


def test_psf_kernel_bitwise(golden):
    g, m, dims, _ = _setup(golden)
    assert np.array_equal(W.gaussian_psf_kernel(dims, float(m["sigma"])).ravel(), g["psf"])


def test_exact_apply_bitwise(golden):
    g, m, dims, basis = _setup(golden)
    op = W.ExactThetaOp(g["psf"].reshape(dims), basis)
    assert np.array_equal(op.apply(g["x0"]), g["exact_apply"])
    assert np.array_equal(op.apply_adjoint(g["x0"]), g["exact_adjoint"])


def test_exact_fista_vs_reference(golden):
    g, m, dims, basis = _setup(golden)
    op = W.ExactThetaOp(g["psf"].reshape(dims), basis)
    I = W.identity_precond(op.n)
    w = W.scale_weights(basis.layout)
    prob = W.DeblurProblem(op, g["x0"], w, m["lambda"])
    tau, it = W.estimate_step(op, I, 1.01, return_iters=True)
    assert abs(tau - m["exact_tau"]) <= 1e-12 * m["exact_tau"]
    # given the reference's tau the iterates are the reference's expressions in fp64
    r = W.fista(prob, I, W.SolverConfig(max_iters=m["iters"], tau=m["exact_tau"], track_energy=True))
    assert r.iters_used == m["exact_iters_used"]
    assert np.array_equal(r.x_final, g["exact_x_final"])  # no reduction touches the iterates
    np.testing.assert_allclose(r.energies, g["exact_energies"], rtol=1e-12)
    r2 = W.fista(prob, I, W.SolverConfig(max_iters=m["iters"], track_energy=False))
    assert abs(r2.tau - m["exact_tau"]) <= 1e-12 * m["exact_tau"]
    assert np.linalg.norm(r2.x_final - g["exact_x_final"]) <= 1e-10 * np.linalg.norm(g["exact_x_final"])
