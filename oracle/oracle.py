"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes binding of the plain-C restatement (oracle/wbx_oracle.c -> oracle/_ref/liboracle.so).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import math
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "liboracle.so"


def build() -> Path:
    """Compile the restatement (gcc only; no /root/reference needed)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "restatement"], check=True)
    return LIB


def _load():
    if not LIB.exists():
        build()
    lib = C.CDLL(str(LIB))
    D = C.POINTER(C.c_double)
    U64 = C.POINTER(C.c_uint64)
    U32 = C.POINTER(C.c_uint32)
    lib.wbxo_filters.argtypes = [C.c_uint32, C.c_uint32, D, D, U32]
    lib.wbxo_analyze.argtypes = [C.c_uint32, U64, C.c_uint32, D, D, C.c_uint32, D, D]
    lib.wbxo_synthesize.argtypes = [C.c_uint32, U64, C.c_uint32, D, D, C.c_uint32, D, D]
    lib.wbxo_spmv.argtypes = [C.c_void_p, D, D]
    lib.wbxo_transpose.argtypes = [C.c_void_p, U64, U32, D]
    lib.wbxo_prox.argtypes = [C.c_uint64, D, C.c_double, D, C.c_double, D, D]
    lib.wbxo_energy.argtypes = [C.c_void_p, D, D, D, C.c_double, C.c_uint64]
    lib.wbxo_energy.restype = C.c_double
    lib.wbxo_estimate_step.argtypes = [C.c_void_p, C.c_void_p, D, C.c_double, U32]
    lib.wbxo_estimate_step.restype = C.c_double
    lib.wbxo_pgd.argtypes = [C.c_void_p, C.c_void_p, D, D, C.c_double, D, C.c_uint64, C.c_double,
                             C.c_double, C.c_double, C.c_int, C.c_int, D, D, U64, D, D]
    lib.wbxo_pgd_tau.argtypes = [C.c_void_p, C.c_void_p, D, D, C.c_double, D, C.c_double, C.c_uint64,
                                 C.c_int, C.c_int, D]
    lib.wbxo_gram_diagonals.argtypes = [C.c_void_p, C.c_uint64, D, D]
    lib.wbxo_spai.argtypes = [C.c_void_p, D]
    lib.wbxo_jacobi.argtypes = [C.c_void_p, C.c_double, D]
    lib.wbxo_rng_normals.argtypes = [C.c_uint64, C.c_uint64, D]
    lib.wbxo_rng_uniforms.argtypes = [C.c_uint64, C.c_uint64, D]
    return lib


lib = _load()


class _Csr(C.Structure):
    _fields_ = [("n", C.c_uint64), ("row_offsets", C.POINTER(C.c_uint64)),
                ("col_indices", C.POINTER(C.c_uint32)), ("values", C.POINTER(C.c_double))]


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Csr:
    """Keeps the numpy arrays alive behind a wbxo_csr view."""

    def __init__(self, n, row_offsets, col_indices, values):
        self.n = int(n)
        self.ro = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        self.ci = np.ascontiguousarray(col_indices, dtype=np.uint32)
        self.va = np.ascontiguousarray(values, dtype=np.float64)
        self.s = _Csr(self.n, self.ro.ctypes.data_as(C.POINTER(C.c_uint64)),
                      self.ci.ctypes.data_as(C.POINTER(C.c_uint32)), _d(self.va))

    @property
    def ptr(self):
        return C.byref(self.s)

    @staticmethod
    def of(op) -> "Csr":
        return Csr(op.n, op.row_offsets, op.col_indices, op.values)

    def transpose(self) -> "Csr":
        nnz = self.va.size
        to = np.zeros(self.n + 1, dtype=np.uint64)
        ti = np.zeros(max(nnz, 1), dtype=np.uint32)
        tv = np.zeros(max(nnz, 1), dtype=np.float64)
        lib.wbxo_transpose(self.ptr, to.ctypes.data_as(C.POINTER(C.c_uint64)),
                           ti.ctypes.data_as(C.POINTER(C.c_uint32)), _d(tv))
        return Csr(self.n, to, ti[:nnz], tv[:nnz])


def filters(family: int, order: int):
    lo, hi = np.zeros(20), np.zeros(20)
    ln = C.c_uint32()
    st = lib.wbxo_filters(family, order, _d(lo), _d(hi), C.byref(ln))
    if st != 0:
        raise ValueError("unsupported filter")
    return lo[: ln.value].copy(), hi[: ln.value].copy()


def _dims(dims):
    return np.array(dims, dtype=np.uint64)


def analyze(u, dims, J, family, order):
    lo, hi = filters(family, order)
    d = _dims(dims)
    u = np.ascontiguousarray(u, dtype=np.float64).ravel()
    x = np.empty(u.size)
    st = lib.wbxo_analyze(len(dims), d.ctypes.data_as(C.POINTER(C.c_uint64)), J, _d(lo), _d(hi),
                          lo.size, _d(u), _d(x))
    assert st == 0
    return x


def synthesize(x, dims, J, family, order):
    lo, hi = filters(family, order)
    d = _dims(dims)
    x = np.ascontiguousarray(x, dtype=np.float64)
    u = np.empty(x.size)
    st = lib.wbxo_synthesize(len(dims), d.ctypes.data_as(C.POINTER(C.c_uint64)), J, _d(lo), _d(hi),
                             lo.size, _d(x), _d(u))
    assert st == 0
    return u


def spmv(A: Csr, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(A.n)
    lib.wbxo_spmv(A.ptr, _d(x), _d(y))
    return y


def prox(z0, tau, w, lam, p):
    z0 = np.ascontiguousarray(z0, dtype=np.float64)
    z = np.empty(z0.size)
    lib.wbxo_prox(z0.size, _d(z0), tau, _d(np.ascontiguousarray(w, dtype=np.float64)), lam,
                  _d(np.ascontiguousarray(p, dtype=np.float64)), _d(z))
    return z


def energy(A: Csr, x, x0, w, lam):
    return lib.wbxo_energy(A.ptr, _d(np.ascontiguousarray(x, dtype=np.float64)),
                           _d(np.ascontiguousarray(x0, dtype=np.float64)),
                           _d(np.ascontiguousarray(w, dtype=np.float64)), lam, A.n)


def estimate_step(A: Csr, AT: Csr, p, step_safety=1.0):
    it = C.c_uint32()
    tau = lib.wbxo_estimate_step(A.ptr, AT.ptr, _d(np.ascontiguousarray(p, dtype=np.float64)),
                                 step_safety, C.byref(it))
    return tau, it.value


def pgd(A: Csr, AT: Csr, x0, w, lam, p, max_iters, accelerate=True, zero_momentum=False,
        step_safety=1.01, rel_energy_tol=1e-3, ref_energy=math.nan, energies=False):
    n = A.n
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    xf = np.empty(n)
    en = np.zeros(max(int(max_iters), 1))
    used = C.c_uint64()
    tau = C.c_double()
    e0 = C.c_double()
    st = lib.wbxo_pgd(A.ptr, AT.ptr, _d(x0), _d(np.ascontiguousarray(w, dtype=np.float64)), lam,
                      _d(np.ascontiguousarray(p, dtype=np.float64)), int(max_iters), rel_energy_tol,
                      step_safety, ref_energy, int(zero_momentum), int(accelerate), _d(xf),
                      _d(en) if energies else None, C.byref(used), C.byref(tau), C.byref(e0))
    if st != 0:
        raise RuntimeError(f"oracle pgd status {st}")
    return dict(x_final=xf, iters_used=used.value, tau=tau.value, initial_energy=e0.value,
                energies=en[: used.value] if energies else None)


def pgd_tau(A: Csr, AT: Csr, x0, w, lam, p, tau, max_iters, accelerate=True, zero_momentum=False):
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    xf = np.empty(A.n)
    st = lib.wbxo_pgd_tau(A.ptr, AT.ptr, _d(x0), _d(np.ascontiguousarray(w, dtype=np.float64)), lam,
                          _d(np.ascontiguousarray(p, dtype=np.float64)), tau, int(max_iters),
                          int(zero_momentum), int(accelerate), _d(xf))
    assert st == 0
    return xf


def gram_diagonals(A: Csr, cap=50):
    m, m2 = np.empty(A.n), np.empty(A.n)
    st = lib.wbxo_gram_diagonals(A.ptr, cap, _d(m), _d(m2))
    return m, m2, st


def spai(A: Csr):
    p = np.empty(A.n)
    assert lib.wbxo_spai(A.ptr, _d(p)) == 0
    return p


def jacobi(A: Csr, eps):
    p = np.empty(A.n)
    assert lib.wbxo_jacobi(A.ptr, eps, _d(p)) == 0
    return p


def rng_normals(seed, n):
    out = np.empty(n)
    lib.wbxo_rng_normals(seed, n, _d(out))
    return out
