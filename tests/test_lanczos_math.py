"""CPU check of the identity behind the Lanczos step estimate (csrc/lanczos.cuh,
tau_lanczos_win_kernel): the reference's power iteration (solver.cpp:69-99) run on M from v0
and the same power iteration run on the Lanczos tridiagonal T_m from e1 give the same
lambda sequence, hence the same stopping index and tau, once m is large enough (exactly for
every iteration it with 2it+1 <= 2m-1; numerically far earlier). Pure numpy, fp64."""
import numpy as np
import pytest


def power_lambdas(M, v0, n_it=200):
    v = v0 / np.linalg.norm(v0)
    out = []
    for _ in range(n_it):
        w = M @ v
        out.append(v @ w)
        v = w / np.linalg.norm(w)
    return np.array(out)


def lanczos(M, v0, m):
    q, qp, beta = v0 / np.linalg.norm(v0), np.zeros_like(v0), 0.0
    al, be = [], []
    for _ in range(m):
        w = M @ q - beta * qp
        a = q @ w
        w -= a * q
        beta = np.linalg.norm(w)
        al.append(a)
        be.append(beta)
        qp, q = q, w / beta
    return np.array(al), np.array(be[:-1])


def tridiagonal_lambdas(al, be, n_it=200):
    """the kernel's formulation: y = T^(2it) e1 / mu_2it, lambda_it = alpha_0 + beta_1 y_1,
    one product by the pentadiagonal T^2 per iteration"""
    T = np.diag(al) + np.diag(be, 1) + np.diag(be, -1)
    T2 = T @ T
    y = np.zeros(len(al))
    y[0] = 1.0
    out = []
    for _ in range(n_it):
        out.append(al[0] + (be[0] * y[1] if len(al) > 1 else 0.0))
        z = T2 @ y
        y = z / z[0]
    return np.array(out)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tridiagonal_power_iteration_reproduces_lambda_sequence(seed):
    rng = np.random.default_rng(seed)
    n = 400
    # clustered top of the spectrum, like a blur operator's low frequencies
    ev = np.concatenate([1.0 - 0.02 * rng.random(40), 0.9 * rng.random(n - 40)])
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    M = (Q * ev) @ Q.T
    v0 = rng.standard_normal(n)
    ref = power_lambdas(M, v0)
    al, be = lanczos(M, v0, 100)   # 2*199+1 <= 2*100-1 does not hold: numerical convergence
    got = tridiagonal_lambdas(al, be)
    assert np.max(np.abs(got - ref) / ref) < 1e-12
    # and the estimate converges well before m = 100
    al60, be60 = lanczos(M, v0, 60)
    assert abs(tridiagonal_lambdas(al60, be60)[-1] - ref[-1]) <= 1e-9 * ref[-1]


def test_small_krylov_space_is_exact():
    """three distinct eigenvalues: Lanczos breaks down after 3 steps and T_3 is exact"""
    rng = np.random.default_rng(3)
    n = 50
    ev = rng.choice([0.5, 1.0, 2.0], n)
    M = np.diag(ev)
    v0 = rng.standard_normal(n)
    al, be = lanczos(M, v0, 3)
    assert np.allclose(tridiagonal_lambdas(al, be), power_lambdas(M, v0), rtol=1e-13, atol=0)
