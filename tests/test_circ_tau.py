"""Block-Fourier step estimate (csrc/circ_tau.cu) on the device, through the C ABI.

For a translation-invariant Theta_K (whole circulant generator groups kept) and a
preconditioner constant on the translation orbits, the fp32 hot path computes the
reference's estimate_step (solver.cpp:69-99) as NG independent power iterations on the
nCo x nCo Fourier blocks of M = P^-1/2 Theta^T Theta P^-1/2. Bar: tau within 1e-12 of the
reference's (fp64 rounding; the full-operator fp32 Lanczos estimate is ~2e-8 off) and the
reference's iteration count. Operators that are not invariant keep the Lanczos estimate."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_08401_b200 import waveblur as W
from paper_1512_08401_b200._native import lib

pytestmark = pytest.mark.gpu

INVARIANT = ["c1_db4_256", "c1_sym6_256", "s64_sym6_ista", "c2_db4_1024"]
NOT_INVARIANT = ["s32_sym4_naive", "s64_sym6_spai", "s128_1d_sym6"]


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


def circ_info(op, dims, J):
    info = (C.c_uint32 * 5)()
    why = C.create_string_buffer(256)
    d = np.array(list(dims) + [1] * (2 - len(dims)), dtype=np.uint64)
    st = lib.wbx_diag_circ_info(op.device(), len(dims), d.ctypes.data_as(C.POINTER(C.c_uint64)), J, info, why, 256)
    assert st == 0
    return list(info), why.value.decode()


def deblurrer(g, op, P, iters=0, precision=32):
    return W.Deblurrer(op, basis_of(g), P, g.weights(), g.meta["lambda"],
                       W.SolverConfig(max_iters=iters, precision=precision, track_energy=False))


@pytest.mark.parametrize("name", INVARIANT)
def test_circ_tau_vs_reference(golden, name):
    g = golden(name)
    op = g.operator()
    info, why = circ_info(op, g.dims, g.meta["J"])
    assert info[0] == 1, why
    P = precond_of(g, op)
    d = deblurrer(g, op, P, iters=2)
    assert d.kernels()[0] == "circ_lanczos_kernel"
    _, rep = d.deblur(np.zeros(g.dims), clamp=False)  # tau does not depend on the image
    assert abs(rep.tau - g.meta["tau"]) <= 1e-12 * g.meta["tau"], (rep.tau, g.meta["tau"])
    A = O.Csr.of(op)
    _, it_ref = O.estimate_step(A, A.transpose(), P.p, 1.01)
    assert rep.tau_iters == it_ref
    assert d.tau_stats()[2] == 0  # no full-operator products


@pytest.mark.parametrize("name", NOT_INVARIANT)
def test_not_invariant_keeps_lanczos(golden, name):
    g = golden(name)
    op = g.operator()
    info, why = circ_info(op, g.dims, g.meta["J"])
    assert info[0] == 0 and why
    d = deblurrer(g, op, precond_of(g, op))
    assert d.kernels()[0] != "circ_lanczos_kernel"
    _, rep = d.deblur(np.zeros(g.dims), clamp=False)
    assert abs(rep.tau - g.meta["tau"]) <= 1e-6 * g.meta["tau"]


def test_circ_tau_orbit_constant_random_preconditioners(golden):
    """Random preconditioners constant on the translation orbits (the estimate applies) and
    one varying inside an orbit (it must not): tau and iteration count vs the oracle's fp64
    power iteration on the full operator."""
    g = golden("c1_db4_256")
    op = g.operator()
    lay = op.layout
    A = O.Csr.of(op)
    AT = A.transpose()
    g0 = g1 = 256 >> 4
    rng = np.random.default_rng(7)
    for trial in range(4):
        p = np.empty(op.n)
        for b in lay.bands:  # one value per (band, orbit representative)
            s0, s1 = b.shape[0] // g0, b.shape[1] // g1
            vals = rng.uniform(0.3, 3.0, (s0, s1))
            p0, p1 = np.meshgrid(np.arange(b.shape[0]), np.arange(b.shape[1]), indexing="ij")
            p[b.offset:b.offset + b.count()] = vals[p0 % s0, p1 % s1].ravel()
        P = W.DiagonalPreconditioner(p, W.PrecondKind.Spai)
        d = deblurrer(g, op, P)
        assert d.kernels()[0] == "circ_lanczos_kernel"
        _, rep = d.deblur(g["u0"].reshape(g.dims), clamp=False)
        t_ref, it_ref = O.estimate_step(A, AT, p, 1.01)
        assert rep.tau_iters == it_ref, (trial, rep.tau_iters, it_ref)
        assert abs(rep.tau - t_ref) <= 1e-12 * t_ref, (trial, rep.tau, t_ref)
    p[int(op.col_indices.max())] *= 1.5  # a column of Theta off its orbit's representative
    d = deblurrer(g, op, W.DiagonalPreconditioner(p, W.PrecondKind.Spai))
    assert d.kernels()[0] != "circ_lanczos_kernel"


def test_circ_tau_through_fista_without_basis(golden):
    """The drop-in fista() has no basis: the operator's own layout (SparseOperator::layout,
    attached by wbx_op_set_layout) selects the estimate; the result is the reference's tau."""
    g = golden("c1_db4_256")
    op = g.operator()
    P = precond_of(g, op)
    prob = W.DeblurProblem(W.SparseThetaOp(op), np.zeros(op.n), g.weights(), g.meta["lambda"])
    r = W.fista(prob, P, W.SolverConfig(max_iters=0, precision=32, track_energy=False))
    assert abs(r.tau - g.meta["tau"]) <= 1e-12 * g.meta["tau"]


def test_circ_tau_deblur_parity_and_determinism(golden):
    """Full C1 deblur with the block-Fourier tau: restored image within the north_star bar of
    the reference's, bitwise reproducible run to run."""
    g = golden("c1_db4_256")
    op = g.operator()
    d = deblurrer(g, op, precond_of(g, op), iters=g.meta["iters"])
    u1, r1 = d.deblur(g["u0"].reshape(g.dims), clamp=False)
    u2, r2 = d.deblur(g["u0"].reshape(g.dims), clamp=False)
    assert r1.tau == r2.tau and np.array_equal(u1, u2)
    ref = g["restored"].reshape(g.dims)
    assert np.linalg.norm(u1 - ref) / np.linalg.norm(ref) <= 1e-5


def test_circ_tau_identity_operator():
    """Identity Theta on a 2-D layout: invariant, M = P^-1, tau = 1 / (max(1/p) * safety)."""
    dims, J = (64, 64), 2  # g = 16: 16 orbits
    n = 64 * 64
    lay = W.make_layout(dims, J)
    eye = W.SparseOperator(n, np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.uint32), np.ones(n), lay)
    info, why = circ_info(eye, dims, J)
    assert info[0] == 1, why
    b = W.make_basis(W.FilterFamily.Daubechies, 2, dims, J)
    d = W.Deblurrer(eye, b, W.identity_precond(n), W.scale_weights(lay), 1e-4,
                    W.SolverConfig(max_iters=1, track_energy=False, step_safety=1.0))
    _, rep = d.deblur(np.zeros(dims), clamp=False)
    assert d.kernels()[0] == "circ_lanczos_kernel"
    assert abs(rep.tau - 1.0) <= 1e-14
    assert rep.tau_iters == W.estimate_step(W.SparseThetaOp(eye), W.identity_precond(n), 1.0, return_iters=True)[1]
