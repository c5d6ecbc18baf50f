"""The whole device pipeline on shapes the golden fixtures do not cover: rectangular images,
a single decomposition level, Haar and db2 filters, an operator built on the device
(theta_conv_topk), SPAI on the device, then the window-engine deblur (fp32 hot path) and the
bitwise fp64 solve, each against the plain-C oracle on the same operator and inputs."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_08401_b200 import synthetic as S
from paper_1512_08401_b200 import waveblur as W

pytestmark = pytest.mark.gpu

CASES = [  # dims, family, order, J, sigma, K factor
    ((64, 128), W.FilterFamily.Symmlet, 4, 3, 2.0, 3),
    ((128, 32), W.FilterFamily.Daubechies, 2, 2, 1.5, 2),
    ((64, 64), W.FilterFamily.Haar, 1, 1, 3.0, 4),
    ((256,), W.FilterFamily.Daubechies, 4, 4, 2.5, 3),
]


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("dims,fam,order,J,sigma,kf", CASES)
def test_device_pipeline_vs_oracle(dims, fam, order, J, sigma, kf):
    basis = W.make_basis(fam, order, dims, J)
    n = basis.layout.total()
    psf = W.gaussian_psf_kernel(dims, sigma)
    op = W.theta_from_generators(W.theta_conv_topk(basis, psf, kf * n, W.dyadic_band_weights(basis.layout)))
    P = W.spai(op)
    A = O.Csr.of(op)
    AT = A.transpose()
    assert np.array_equal(P.p, O.spai(A))
    clean = S.synthetic_scene(dims)
    u0 = S.add_noise(W.synthesize(W.spmv(op, W.analyze(clean, basis).values), basis), 5e-3, 9)
    w = W.scale_weights(basis.layout)
    fam_i, iters = int(fam), 40
    x0 = O.analyze(u0, dims, J, fam_i, order)
    ref = O.pgd(A, AT, x0, w, 1e-4, P.p, iters)
    u_ref = O.synthesize(ref["x_final"], dims, J, fam_i, order)
    # window-engine fp32 hot path
    d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=iters, track_energy=False))
    u, rep = d.deblur(u0, clamp=False)
    assert abs(rep.tau - ref["tau"]) <= 1e-6 * ref["tau"]
    assert _rel(u.ravel(), u_ref) <= 1e-5
    # fp64 reference mode: bitwise given tau
    prob = W.DeblurProblem(W.SparseThetaOp(op), x0, w, 1e-4)
    r64 = W.fista(prob, P, W.SolverConfig(max_iters=iters, precision=64, tau=ref["tau"], track_energy=False))
    assert np.array_equal(r64.x_final, O.pgd_tau(A, AT, x0, w, 1e-4, P.p, ref["tau"], iters))
