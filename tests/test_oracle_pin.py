"""The oracle (plain-C restatement, oracle/wbx_oracle.c) pinned against the REFERENCE's
own outputs (tests/golden, produced by the unmodified reference via
oracle/make_golden.py). Bitwise wherever the reference's arithmetic is reproducible;
these run on CPU."""
import math

import numpy as np
import pytest

from oracle import oracle as O


CASES = ["c1_db4_256", "c1_sym6_256", "s64_sym6_ista", "s32_sym4_naive", "s64_sym6_spai", "s128_1d_sym6"]


def test_filters_match_reference_invariants():
    # test_wavelet.cpp:21-57
    for fam, order, length in [(0, 1, 2), (1, 2, 4), (1, 10, 20), (2, 4, 8), (2, 6, 12), (2, 8, 16)]:
        lo, hi = O.filters(fam, order)
        assert lo.size == length
        assert abs((lo * lo).sum() - 1.0) < 1e-12
        assert abs(lo.sum() - math.sqrt(2.0)) < 1e-12
        for i in range(length):
            assert hi[i] == (1.0 if i % 2 == 0 else -1.0) * lo[length - 1 - i]


def test_haar_known_answers():
    # test_wavelet.cpp:114-120: analyze([1,1,1,1], Haar, J=2) = [2,0,0,0]
    x = O.analyze(np.ones(4), (4,), 2, 0, 1)
    assert abs(x[0] - 2.0) < 1e-14 and np.all(np.abs(x[1:]) < 1e-14)
    # :131-137 N=2 scaling function
    u = O.synthesize(np.array([1.0, 0.0]), (2,), 1, 0, 1)
    assert np.allclose(u, [1 / math.sqrt(2)] * 2, rtol=0, atol=1e-15)


def test_counter_rng_box_muller_pairs():
    v = O.rng_normals(0x5EED, 5)
    v4 = O.rng_normals(0x5EED, 4)
    assert np.array_equal(v[:4], v4)


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_reference_bitwise(golden, name):
    g = golden(name)
    m = g.meta
    fam, order, J = g.family, m["order"], m["J"]
    op = g.operator()                     # generator list -> CSR (wbx_theta_expand, host)
    assert op.nnz() == m["nnz"]
    A = O.Csr.of(op)
    AT = A.transpose()
    w = g.weights()
    if "u0" in g:
        x0 = O.analyze(g["u0"], g.dims, J, fam, order)
        if "x0" in g:
            assert np.array_equal(x0, g["x0"]), "analyze differs from the reference"
    else:
        pytest.skip("no stored input vector")
    if m["precond"] == "spai":
        p = O.spai(A)
    elif m["precond"] == "jacobi":
        mm, _, _ = O.gram_diagonals(A)
        p = O.jacobi(A, max(1e-3 * mm.max(), 1e-300))
    else:
        p = np.ones(g.n)
    if "p" in g:
        assert np.array_equal(p, g["p"]), "preconditioner differs from the reference"
    r = O.pgd(A, AT, x0, w, m["lambda"], p, m["iters"], accelerate=(m["method"] != "ista"),
              energies=True)
    assert r["tau"] == m["tau"], "estimate_step differs from the reference"
    assert r["initial_energy"] == m["initial_energy"]
    assert np.array_equal(r["x_final"], g["x_final"]), "x_final differs from the reference"
    assert np.array_equal(r["energies"], g["energies"])
    u = O.synthesize(r["x_final"], g.dims, J, fam, order)
    if "restored" in g:
        assert np.array_equal(u, g["restored"]), "synthesize differs from the reference"


def test_oracle_transpose_roundtrip(golden):
    g = golden("s64_sym6_spai")
    A = O.Csr.of(g.operator())
    B = A.transpose().transpose()
    assert np.array_equal(A.ro, B.ro) and np.array_equal(A.ci, B.ci) and np.array_equal(A.va, B.va)
