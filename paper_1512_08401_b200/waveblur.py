"""Python mirror of the reference's C++ hot-path API (waveblur, /root/reference/proj).

Same names, argument meaning and error behaviour as the reference headers
(`include/waveblur/{wavelet,theta,precond,solver}.hpp`); every compute call goes
through the C ABI of libwbx.so (include/wbx.h) onto the B200. Host-side bookkeeping
that the reference also does on the host (layouts, CSR transposition, WTHETA01 file
I/O) is plain numpy here. Nothing in this module falls back to a CPU computation of a
device operation: if libwbx.so (or a GPU) is missing, the call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import struct
from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

import numpy as np

from . import _native as N

lib = N.lib


# ----------------------------------------------------------------------------- errors
# image.hpp:10-36; the status codes of include/wbx.h map 1:1 onto these.
class WaveblurError(Exception):
    pass


class ShapeMismatch(WaveblurError, ValueError):
    pass


class UnsupportedFilter(WaveblurError, ValueError):
    pass


class BandNotFound(WaveblurError, ValueError):
    pass


class BadSpec(WaveblurError, ValueError):
    pass


class TooLarge(WaveblurError, ValueError):
    pass


class BadEpsilon(WaveblurError, ValueError):
    pass


class MemoryGuard(WaveblurError, RuntimeError):
    pass


class NonFiniteEnergy(WaveblurError, RuntimeError):
    pass


class IoError(WaveblurError, RuntimeError):
    pass


class CudaError(WaveblurError, RuntimeError):
    pass


_STATUS = {1: ShapeMismatch, 2: UnsupportedFilter, 3: BandNotFound, 4: BadSpec, 5: TooLarge,
           6: BadEpsilon, 7: MemoryGuard, 8: NonFiniteEnergy, 9: IoError, 10: CudaError,
           11: ValueError}


def _check(status: int) -> None:
    if status != N.WBX_OK:
        raise _STATUS.get(status, WaveblurError)(N.last_error())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u64ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _u32ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _f64(x, n: Optional[int] = None, what: str = "vector") -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if n is not None and a.size != n:
        raise ShapeMismatch(f"{what}: length {a.size} != {n}")
    return a


# ----------------------------------------------------------------------------- device context
class Context:
    """One CUDA device + stream (wbx_ctx). Calls on one context are serialised."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib.wbx_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    @property
    def stream(self) -> int:
        return lib.wbx_ctx_stream(self.handle) or 0

    def synchronize(self) -> None:
        _check(lib.wbx_ctx_synchronize(self.handle))

    @property
    def launches(self) -> int:
        return int(lib.wbx_ctx_launch_count(self.handle))

    def __del__(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        if getattr(self, "handle", None):
            lib.wbx_ctx_destroy(self.handle)
            self.handle = None


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ----------------------------------------------------------------------------- wavelets
class FilterFamily(enum.IntEnum):  # wavelet.hpp:12
    Haar = 0
    Daubechies = 1
    Symmlet = 2


def family_name(f: FilterFamily) -> str:
    return {0: "haar", 1: "daubechies", 2: "symmlet"}[int(f)]


@dataclass
class FilterPair:  # wavelet.hpp:18-28
    family: FilterFamily
    order: int
    lowpass: np.ndarray
    highpass: np.ndarray

    def length(self) -> int:
        return len(self.lowpass)


def make_filters(family: Union[FilterFamily, str], order: Optional[int] = None) -> FilterPair:
    """make_filters (wavelet_filters.cpp:110-161)."""
    if isinstance(family, str):
        f, o = C.c_uint32(), C.c_uint32()
        _check(lib.wbx_parse_filter(family.encode(), C.byref(f), C.byref(o)))
        family, order = FilterFamily(f.value), o.value
    lo = np.zeros(20)
    hi = np.zeros(20)
    ln = C.c_uint32()
    _check(lib.wbx_make_filters(int(family), int(order), _dptr(lo), _dptr(hi), C.byref(ln)))
    return FilterPair(FilterFamily(family), int(order), lo[: ln.value].copy(), hi[: ln.value].copy())


@dataclass
class Band:  # wavelet.hpp:39-52
    level: int
    orientation: int
    shape: tuple
    offset: int

    def count(self) -> int:
        return int(np.prod(self.shape))


@dataclass
class SubbandLayout:  # wavelet.hpp:58-64
    dims: tuple
    J: int
    bands: list

    def total(self) -> int:
        return int(np.prod(self.dims))

    def find(self, level: int, orientation: int) -> Band:
        for b in self.bands:
            if b.level == level and b.orientation == orientation:
                return b
        raise BandNotFound(f"no band (level={level}, e={orientation})")

    def band_of_flat(self, flat: int) -> int:
        for i in range(len(self.bands) - 1, -1, -1):
            if flat >= self.bands[i].offset:
                return i
        raise BandNotFound("flat index out of range")


def make_layout(dims: Sequence[int], J: int) -> SubbandLayout:
    """make_layout (wavelet.cpp:32-70)."""
    dims = tuple(int(d) for d in dims)
    if len(dims) < 1 or len(dims) > 2:
        raise ShapeMismatch("layout needs 1 or 2 dims")
    d = np.array(dims, dtype=np.uint64)
    out = (N.wbx_band * (1 + 3 * max(int(J), 1)))()
    nb = C.c_uint32()
    _check(lib.wbx_make_layout(len(dims), _u64ptr(d), int(J), out, C.byref(nb)))
    bands = []
    for i in range(nb.value):
        b = out[i]
        shape = (int(b.shape[0]), int(b.shape[1])) if len(dims) == 2 else (int(b.shape[0]),)
        bands.append(Band(int(b.level), int(b.orientation), shape, int(b.offset)))
    return SubbandLayout(dims, int(J), bands)


class WaveletBasis:  # wavelet.hpp:68-74, plus its device residency (wbx_basis)
    def __init__(self, filters: FilterPair, layout: SubbandLayout, ctx: Optional[Context] = None):
        self.filters = filters
        self.layout = layout
        self._ctx = ctx
        self._handles = {}  # Context -> native handle

    def dims(self):
        return self.layout.dims

    def levels(self) -> int:
        return self.layout.J

    def device(self, ctx: Optional[Context] = None):
        """The native basis on `ctx`. One handle per context, created on first use and kept
        until this object dies: a solver built on a handle can never see it freed (a later
        call on another context creates a second handle instead of replacing the first)."""
        ctx = ctx or self._ctx or default_context()
        h = self._handles.get(ctx)
        if h is None:
            d = np.array(self.layout.dims, dtype=np.uint64)
            h = C.c_void_p()
            _check(lib.wbx_basis_create(ctx.handle, int(self.filters.family), self.filters.order,
                                        len(self.layout.dims), _u64ptr(d), self.layout.J, C.byref(h)))
            self._handles[ctx] = h
            if self._ctx is None:
                self._ctx = ctx
        return h

    def _release(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        for h in self._handles.values():
            lib.wbx_basis_destroy(h)
        self._handles.clear()

    def __del__(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        self._release()


def make_basis(family_or_name, *args) -> WaveletBasis:
    """make_basis (wavelet.cpp:72-80): (family, order, dims, J) or (name, dims, J)."""
    if isinstance(family_or_name, str):
        dims, J = args
        return WaveletBasis(make_filters(family_or_name), make_layout(dims, J))
    order, dims, J = args
    return WaveletBasis(make_filters(family_or_name, order), make_layout(dims, J))


@dataclass
class WaveletCoeffs:  # wavelet.hpp:81-84
    layout: SubbandLayout
    values: np.ndarray


def analyze(signal: np.ndarray, basis: WaveletBasis, ctx: Optional[Context] = None) -> WaveletCoeffs:
    """x = Psi^* u (wavelet.cpp:254-256), on the device, bitwise equal to the reference."""
    u = np.asarray(signal, dtype=np.float64)
    if tuple(u.shape) != tuple(basis.layout.dims):
        raise ShapeMismatch("signal dims do not match basis")
    ctx = ctx or basis._ctx or default_context()
    u = np.ascontiguousarray(u).ravel()
    x = np.empty(u.size)
    _check(lib.wbx_analyze(ctx.handle, basis.device(ctx), _dptr(u), _dptr(x)))
    return WaveletCoeffs(basis.layout, x)


def synthesize(coeffs: Union[WaveletCoeffs, np.ndarray], basis: WaveletBasis,
               ctx: Optional[Context] = None) -> np.ndarray:
    """u = Psi x (wavelet.cpp:258-260), on the device, bitwise equal to the reference."""
    vals = coeffs.values if isinstance(coeffs, WaveletCoeffs) else coeffs
    x = _f64(vals)
    if x.size != basis.layout.total():
        raise ShapeMismatch("coefficient length does not match basis")
    ctx = ctx or basis._ctx or default_context()
    u = np.empty(x.size)
    _check(lib.wbx_synthesize(ctx.handle, basis.device(ctx), _dptr(x), _dptr(u)))
    return u.reshape(basis.layout.dims)


def single_wavelet(basis: WaveletBasis, level: int, orientation: int,
                   ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or basis._ctx or default_context()
    u = np.empty(basis.layout.total())
    _check(lib.wbx_single_wavelet(ctx.handle, basis.device(ctx), level, orientation, _dptr(u)))
    return u.reshape(basis.layout.dims)


# ----------------------------------------------------------------------------- Theta_K
class SparseOperator:
    """K-sparse CSR operator (theta.hpp:50-60): u64 row offsets, u32 strictly increasing
    columns per row, f64 values, plus subband metadata. Device layouts are built lazily
    on first use (wbx_op_create) and cached per context."""

    def __init__(self, n: int, row_offsets, col_indices, values, layout: Optional[SubbandLayout] = None,
                 family: FilterFamily = FilterFamily.Haar, order: int = 1):
        self.n = int(n)
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        self.col_indices = np.ascontiguousarray(col_indices, dtype=np.uint32)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.layout = layout
        self.family = FilterFamily(family)
        self.order = int(order)
        self._devs = {}  # Context -> native handle
        self._ctx = None

    def nnz(self) -> int:
        return int(self.values.size)

    def device(self, ctx: Optional[Context] = None):
        """The device layouts on `ctx` (wbx_op_create). One handle per context, kept until
        this object dies, so solvers and Deblurrers built on a handle never see it freed."""
        ctx = ctx or self._ctx or default_context()
        h = self._devs.get(ctx)
        if h is None:
            if self.row_offsets.size != self.n + 1:
                raise ShapeMismatch("row_offsets must have n+1 entries")
            h = C.c_void_p()
            _check(lib.wbx_op_create(ctx.handle, self.n, _u64ptr(self.row_offsets),
                                     _u32ptr(self.col_indices), _dptr(self.values), C.byref(h)))
            if self.layout is not None:  # SparseOperator::layout (theta.hpp:55)
                d = np.array(self.layout.dims, dtype=np.uint64)
                st = lib.wbx_op_set_layout(h, len(self.layout.dims), _u64ptr(d), self.layout.J)
                if st != N.WBX_OK:
                    lib.wbx_op_destroy(h)
                    _check(st)
            gl = getattr(self, "generators", None)
            if gl is not None:
                d = np.array(gl.dims, dtype=np.uint64)
                st = lib.wbx_op_set_generators(h, len(gl.dims), _u64ptr(d), gl.J, gl.blocks.size, _u32ptr(gl.blocks),
                                               _u32ptr(gl.gen_index), _u64ptr(gl.counts), _dptr(gl.values))
                if st != N.WBX_OK:
                    lib.wbx_op_destroy(h)
                    _check(st)
            self._devs[ctx] = h
            if self._ctx is None:
                self._ctx = ctx
        return h

    def info(self, ctx: Optional[Context] = None) -> N.wbx_op_info:
        inf = N.wbx_op_info()
        _check(lib.wbx_op_get_info(self.device(ctx), C.byref(inf)))
        return inf

    def _release(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        for h in self._devs.values():
            lib.wbx_op_destroy(h)
        self._devs.clear()

    def __del__(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        self._release()


def _ctx_of(op: SparseOperator, ctx):
    return ctx or op._ctx or default_context()


def spmv(op: SparseOperator, x, ctx: Optional[Context] = None) -> np.ndarray:
    """y = Theta_K x (theta.cpp:300-311); fp64, bitwise equal to the reference."""
    xv = _f64(x)
    if xv.size != op.n:
        raise ShapeMismatch("spmv: vector length mismatch")
    ctx = _ctx_of(op, ctx)
    y = np.empty(op.n)
    _check(lib.wbx_spmv(ctx.handle, op.device(ctx), 0, _dptr(xv), _dptr(y)))
    return y


def spmv_t(op: SparseOperator, x, ctx: Optional[Context] = None) -> np.ndarray:
    """y = Theta_K^T x (theta.cpp:344-356)."""
    xv = _f64(x)
    if xv.size != op.n:
        raise ShapeMismatch("spmv_t: vector length mismatch")
    ctx = _ctx_of(op, ctx)
    y = np.empty(op.n)
    _check(lib.wbx_spmv(ctx.handle, op.device(ctx), 1, _dptr(xv), _dptr(y)))
    return y


def approx_gradient(op: SparseOperator, x, x0, ctx: Optional[Context] = None) -> np.ndarray:
    """Theta^T (Theta x - x0) (theta.cpp:358-365)."""
    xv, x0v = _f64(x), _f64(x0)
    if xv.size != op.n or x0v.size != op.n:
        raise ShapeMismatch("approx_gradient: vector length mismatch")
    ctx = _ctx_of(op, ctx)
    g = np.empty(op.n)
    _check(lib.wbx_approx_gradient(ctx.handle, op.device(ctx), _dptr(xv), _dptr(x0v), _dptr(g)))
    return g


def ops_per_pixel(op: SparseOperator) -> float:
    return 2.0 * op.nnz() / op.n


def transpose(op: SparseOperator) -> SparseOperator:
    """Theta_K^T as CSR (theta.cpp:371-382; make_transpose order :324-340). Host-side setup."""
    n = op.n
    cols = op.col_indices.astype(np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(op.row_offsets.astype(np.int64)))
    order = np.lexsort((rows, cols))  # by column, then ascending row (stable CSR scan)
    counts = np.bincount(cols, minlength=n)
    off = np.zeros(n + 1, dtype=np.uint64)
    off[1:] = np.cumsum(counts)
    return SparseOperator(n, off, rows[order].astype(np.uint32), op.values[order], op.layout,
                          op.family, op.order)


def write_operator(op: SparseOperator, path: str) -> None:
    """write_operator (theta.cpp:428-443): the bit-exact WTHETA01 file, through the C ABI."""
    if op.layout is None:
        raise IoError("operator has no layout")
    d = np.array(op.layout.dims, dtype=np.uint64)
    _check(lib.wbx_write_operator(str(path).encode(), len(op.layout.dims), _u64ptr(d), op.layout.J, int(op.family),
                                  op.order, op.n, _u64ptr(op.row_offsets), _u32ptr(op.col_indices),
                                  _dptr(op.values)))


def read_operator(path: str) -> SparseOperator:
    """read_operator (theta.cpp:445-490) with the reference's validation, through the C ABI."""
    nd, J, fam, order = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
    dims = np.zeros(2, dtype=np.uint64)
    n, nnz = C.c_uint64(), C.c_uint64()
    ro, ci, va = _U64P(), _U32P(), _DP()
    _check(lib.wbx_read_operator(str(path).encode(), C.byref(nd), _u64ptr(dims), C.byref(J), C.byref(fam),
                                 C.byref(order), C.byref(n), C.byref(nnz), C.byref(ro), C.byref(ci), C.byref(va)))
    try:
        k = int(nnz.value)
        row_offsets = np.ctypeslib.as_array(ro, shape=(n.value + 1,)).copy()
        cols = np.ctypeslib.as_array(ci, shape=(max(k, 1),))[:k].copy()
        vals = np.ctypeslib.as_array(va, shape=(max(k, 1),))[:k].copy()
    finally:
        lib.wbx_free(ro)
        lib.wbx_free(ci)
        lib.wbx_free(va)
    layout = make_layout([int(v) for v in dims[: nd.value]], J.value)
    return SparseOperator(int(n.value), row_offsets, cols, vals, layout, FilterFamily(fam.value), order.value)


_U64P = lambda: C.POINTER(C.c_uint64)()  # noqa: E731
_U32P = lambda: C.POINTER(C.c_uint32)()  # noqa: E731
_DP = lambda: C.POINTER(C.c_double)()  # noqa: E731


def save_device_operator(op: SparseOperator, path: str, P: Optional["DiagonalPreconditioner"] = None,
                         tau: float = 0.0, ctx: Optional[Context] = None) -> None:
    """Device-ready operator cache (WBXOP001, include/wbx.h wbx_op_save): the device layouts
    (and the window layouts solvers built on `ctx`), optionally P and tau."""
    p = _f64(P.p, op.n, "preconditioner") if P is not None else None
    _check(lib.wbx_op_save(op.device(ctx), str(path).encode(), _dptr(p) if p is not None else None, float(tau)))


def load_device_operator(path: str, ctx: Optional[Context] = None, layout: Optional[SubbandLayout] = None):
    """wbx_op_load: (SparseOperator with its device handle bound to ctx, P or None, tau)."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    inf = N.wbx_op_info()
    # the element count is needed for p before loading: read it from the header
    with open(path, "rb") as f:
        head = f.read(20)
    if len(head) < 20 or head[:8] != b"WBXOP001":
        raise IoError(f"{path}: not a WBXOP001 device operator cache")
    n = struct.unpack_from("<Q", head, 12)[0]
    p = np.empty(n)
    has_p, tau = C.c_int(), C.c_double()
    _check(lib.wbx_op_load(ctx.handle, str(path).encode(), C.byref(h), _dptr(p), C.byref(has_p), C.byref(tau)))
    try:
        _check(lib.wbx_op_get_info(h, C.byref(inf)))
        ro = np.empty(int(inf.n) + 1, dtype=np.uint64)
        ci = np.empty(max(int(inf.nnz), 1), dtype=np.uint32)
        va = np.empty(max(int(inf.nnz), 1), dtype=np.float64)
        _check(lib.wbx_op_get_csr(h, _u64ptr(ro), _u32ptr(ci), _dptr(va)))
    except Exception:
        lib.wbx_op_destroy(h)
        raise
    k = int(inf.nnz)
    op = SparseOperator(int(inf.n), ro, ci[:k], va[:k], layout)
    op._devs[ctx] = h  # the loaded device layouts ARE this operator's handle on ctx
    op._ctx = ctx
    return op, (DiagonalPreconditioner(p, PrecondKind.Spai) if has_p.value else None), float(tau.value)


@dataclass
class GeneratorList:
    """A thresholded circulant Theta_K in compressed form: the kept (block, generator
    index, count, value) groups of the reference's global top-K walk
    (theta.cpp:206-276). block = out_band * nbands + in_band."""
    dims: tuple
    J: int
    family: FilterFamily
    order: int
    blocks: np.ndarray
    gen_index: np.ndarray
    counts: np.ndarray
    values: np.ndarray

    @staticmethod
    def from_bytes(raw: bytes, dims, J, family, order) -> "GeneratorList":
        rec = np.frombuffer(raw, dtype=np.dtype([("b", "<u4"), ("g", "<u4"), ("c", "<u8"), ("v", "<f8")]))
        return GeneratorList(tuple(dims), int(J), FilterFamily(family), int(order),
                             rec["b"].astype(np.uint32), rec["g"].astype(np.uint32),
                             rec["c"].astype(np.uint64), rec["v"].astype(np.float64))

    def to_bytes(self) -> bytes:
        rec = np.zeros(self.blocks.size, dtype=np.dtype([("b", "<u4"), ("g", "<u4"), ("c", "<u8"), ("v", "<f8")]))
        rec["b"], rec["g"], rec["c"], rec["v"] = self.blocks, self.gen_index, self.counts, self.values
        return rec.tobytes()


def theta_from_generators(gl: GeneratorList) -> SparseOperator:
    """Expand a GeneratorList into the CSR the reference's threshold_* would assemble
    (walk theta.cpp:236-275 + assemble :180-201), via wbx_theta_expand."""
    dims = np.array(gl.dims, dtype=np.uint64)
    nnz = C.c_uint64()
    args = (len(gl.dims), _u64ptr(dims), gl.J, gl.blocks.size, _u32ptr(gl.blocks), _u32ptr(gl.gen_index),
            _u64ptr(gl.counts), _dptr(gl.values), C.byref(nnz))
    _check(lib.wbx_theta_expand(*args, None, None, None))
    layout = make_layout(gl.dims, gl.J)
    n = layout.total()
    ro = np.zeros(n + 1, dtype=np.uint64)
    ci = np.zeros(max(nnz.value, 1), dtype=np.uint32)
    va = np.zeros(max(nnz.value, 1), dtype=np.float64)
    _check(lib.wbx_theta_expand(*args, _u64ptr(ro), _u32ptr(ci), _dptr(va)))
    op = SparseOperator(n, ro, ci[: nnz.value], va[: nnz.value], layout, gl.family, gl.order)
    op.generators = gl  # the compressed form: attached to the device operator (stencil engine)
    return op


def gaussian_psf_kernel(dims, sigma: float) -> np.ndarray:
    """generate_psf(GaussianSpec{sigma}, dims).kernel (operators.cpp:100-120, 298-318), with the
    reference's expressions (host libm exp), as the row-major kernel image."""
    d = np.array(dims, dtype=np.uint64)
    k = np.zeros(int(np.prod(dims)), dtype=np.float64)
    _check(lib.wbx_psf_gaussian(len(dims), _u64ptr(d), float(sigma), _dptr(k)))
    return k.reshape(dims)


# ----------------------------------------------------------------------------- PSFs (operators.hpp:15-77)
@dataclass
class GaussianSpec:
    sigma: float


@dataclass
class SkewedGaussianSpec:
    sigma: float


@dataclass
class MotionSpec:
    points: int = 5
    sigma1: float = 8.0  # std-dev of the control point cloud
    sigma2: float = 1.0  # post-smoothing Gaussian
    seed: int = 0


@dataclass
class AirySpec:
    scale: float


@dataclass
class DefocusSpec:
    radius: float


def psf_spec_string(spec) -> str:
    """psf_spec_string (operators.cpp:276-296)."""
    g = lambda v: f"{v:g}"  # noqa: E731  (std::ostream default format)
    if isinstance(spec, GaussianSpec):
        return f"gaussian:{g(spec.sigma)}"
    if isinstance(spec, SkewedGaussianSpec):
        return f"skewed:{g(spec.sigma)}"
    if isinstance(spec, MotionSpec):
        return f"motion:{spec.points}:{g(spec.sigma1)}:{g(spec.sigma2)}:{spec.seed}"
    if isinstance(spec, AirySpec):
        return f"airy:{g(spec.scale)}"
    return f"defocus:{g(spec.radius)}"


@dataclass
class Psf:  # operators.hpp:38-42
    kernel: np.ndarray
    spec: object


def _psf_params(spec):
    if isinstance(spec, GaussianSpec):
        return N.WBX_PSF_GAUSSIAN, [spec.sigma]
    if isinstance(spec, SkewedGaussianSpec):
        return N.WBX_PSF_SKEWED, [spec.sigma]
    if isinstance(spec, MotionSpec):
        return N.WBX_PSF_MOTION, [float(spec.points), spec.sigma1, spec.sigma2, float(spec.seed)]
    if isinstance(spec, AirySpec):
        return N.WBX_PSF_AIRY, [spec.scale]
    if isinstance(spec, DefocusSpec):
        return N.WBX_PSF_DEFOCUS, [spec.radius]
    raise BadSpec("unknown PSF spec")


def generate_psf(spec, dims, ctx: Optional[Context] = None) -> Psf:
    """generate_psf (operators.cpp:298-318): the kernel image (centred at 0, wrap-around, unit
    mass). Motion kernels smooth on the device (their context: ctx or the default)."""
    kind, params = _psf_params(spec)
    dims = tuple(int(d) for d in dims)
    if kind == N.WBX_PSF_MOTION and spec.seed >= 2 ** 53:
        raise BadSpec("motion seed must be < 2^53")
    d = np.array(dims, dtype=np.uint64)
    k = np.zeros(int(np.prod(dims)) if dims else 1, dtype=np.float64)
    c = (ctx or default_context()) if kind == N.WBX_PSF_MOTION else ctx
    _check(lib.wbx_generate_psf(c.handle if c else None, kind, _dptr(np.array(params, dtype=np.float64)), len(dims),
                                _u64ptr(d), _dptr(k)))
    return Psf(k.reshape(dims), spec)


def _kernel_of(psf) -> np.ndarray:
    return np.ascontiguousarray(psf.kernel if isinstance(psf, Psf) else psf, dtype=np.float64)


def _conv(u, psf, adjoint: int, ctx) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    k = _kernel_of(psf)
    if k.shape != u.shape:
        raise ShapeMismatch("convolve: image and kernel dims differ")
    ctx = ctx or default_context()
    out = np.empty_like(u)
    d = np.array(u.shape, dtype=np.uint64)
    _check(lib.wbx_convolve(ctx.handle, u.ndim, _u64ptr(d), _dptr(k), _dptr(u), adjoint, _dptr(out)))
    return out


def convolve(u, psf, ctx: Optional[Context] = None) -> np.ndarray:
    """convolve (operators.cpp:320-322): circular convolution via the device FFT."""
    return _conv(u, psf, 0, ctx)


def apply_adjoint_psf(u, psf, ctx: Optional[Context] = None) -> np.ndarray:
    """apply_adjoint (operators.cpp:324-326): H* u = h~ * u, h~[i] = h[-i]."""
    return _conv(u, psf, 1, ctx)


def add_noise(u, sigma: float, seed: int, ctx: Optional[Context] = None) -> np.ndarray:
    """add_noise (operators.cpp:344-356): per-index Box-Muller, on the device."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    ctx = ctx or default_context()
    out = np.empty_like(u)
    _check(lib.wbx_add_noise(ctx.handle, u.size, _dptr(u), float(sigma), int(seed), _dptr(out)))
    return out


@dataclass
class DegradationModel:  # operators.hpp:69-73
    psf: Psf
    noise_sigma: float = 0.0
    seed: int = 0


def degrade(u, model: DegradationModel, ctx: Optional[Context] = None) -> np.ndarray:
    """degrade (operators.cpp:385-387) = add_noise(convolve(u, psf), sigma, seed), on the device."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    k = _kernel_of(model.psf)
    if k.shape != u.shape:
        raise ShapeMismatch("degrade: image and kernel dims differ")
    ctx = ctx or default_context()
    out = np.empty_like(u)
    d = np.array(u.shape, dtype=np.uint64)
    _check(lib.wbx_degrade(ctx.handle, u.ndim, _u64ptr(d), _dptr(k), _dptr(u), float(model.noise_sigma),
                           int(model.seed), _dptr(out)))
    return out


def dyadic_band_weights(layout: SubbandLayout) -> np.ndarray:
    """Per-band sigma of dyadic_weights (theta.cpp:153-165): 2^(level - J)."""
    return np.array([2.0 ** (b.level - layout.J) for b in layout.bands], dtype=np.float64)


def theta_conv_topk(basis: WaveletBasis, psf_kernel, K: int, band_weights=None, ctx: Optional[Context] = None,
                    max_records: int = 1 << 20) -> GeneratorList:
    """build_theta_conv (theta.cpp:40-79) + threshold_weighted / threshold_naive
    (theta.cpp:206-296) ON THE DEVICE, returned in compressed form (the kept generator
    groups; expand with theta_from_generators). band_weights: per band (default all ones =
    threshold_naive; dyadic_band_weights(...) = threshold_weighted with dyadic_weights)."""
    ctx = ctx or default_context()
    layout = basis.layout
    nb = len(layout.bands)
    w = np.ones(nb) if band_weights is None else np.asarray(band_weights, dtype=np.float64)
    if w.size != nb:
        raise ShapeMismatch("theta_conv_topk: one weight per band")
    psf = _f64(np.asarray(psf_kernel, dtype=np.float64).ravel(), layout.total(), "psf kernel")
    blocks = np.zeros(max_records, dtype=np.uint32)
    gidx = np.zeros(max_records, dtype=np.uint32)
    cnt = np.zeros(max_records, dtype=np.uint64)
    val = np.zeros(max_records, dtype=np.float64)
    nrec = C.c_uint64()
    _check(lib.wbx_theta_conv_topk(ctx.handle, basis.device(ctx), _dptr(psf), _dptr(w), int(K), max_records,
                                   _u32ptr(blocks), _u32ptr(gidx), _u64ptr(cnt), _dptr(val), C.byref(nrec)))
    m = nrec.value
    return GeneratorList(tuple(layout.dims), layout.J, basis.filters.family, basis.filters.order,
                         blocks[:m].copy(), gidx[:m].copy(), cnt[:m].copy(), val[:m].copy())


class StencilOperator:
    """Theta_K applied straight from its kept generator groups: reads only
    x and y. apply_dev / apply_adjoint_dev take device pointers (float64 or float32)."""

    def __init__(self, gl: GeneratorList, ctx: Optional[Context] = None):
        self._ctx = ctx or default_context()
        self.n = int(np.prod(gl.dims))
        dims = np.array(gl.dims, dtype=np.uint64)
        h = C.c_void_p()
        _check(lib.wbx_stencil_create(self._ctx.handle, len(gl.dims), _u64ptr(dims), gl.J, gl.blocks.size,
                                      _u32ptr(gl.blocks), _u32ptr(gl.gen_index), _u64ptr(gl.counts),
                                      _dptr(gl.values), C.byref(h)))
        self.handle = h

    def spmv_dev(self, x_ptr: int, y_ptr: int, transpose: bool = False, precision: int = N.WBX_FP64) -> None:
        _check(lib.wbx_stencil_spmv_dev(self.handle, int(transpose), int(precision), C.c_void_p(x_ptr),
                                        C.c_void_p(y_ptr)))

    def __del__(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        if getattr(self, "handle", None):
            lib.wbx_stencil_destroy(self.handle)
            self.handle = None


@dataclass
class SigmaLadder:
    """Stationary Gaussian Theta_K operators at increasing sigmas (one GeneratorList each)."""
    sigmas: np.ndarray
    levels: list   # [GeneratorList]

    @staticmethod
    def from_npz(z, dims=None, J=4, family=FilterFamily.Daubechies, order=4) -> "SigmaLadder":
        sig = np.asarray(z["sigmas"], dtype=np.float64)
        meta_dims = tuple(json_dims(z)) if dims is None else tuple(dims)
        lv = []
        for l in range(sig.size):
            lv.append(GeneratorList(meta_dims, J, FilterFamily(family), order,
                                    z[f"l{l}_gen_block"].astype(np.uint32), z[f"l{l}_gen_index"].astype(np.uint32),
                                    z[f"l{l}_gen_count"].astype(np.uint64), z[f"l{l}_gen_value"]))
        return SigmaLadder(sig, lv)


def rescale_generators(gl: GeneratorList, new_dims) -> GeneratorList:
    """Carry a thresholded stationary operator to a larger grid (BASELINE config C4: the
    4096^2 operators are derived from the reference's 1024^2 ones). A generator entry is a
    circular offset on its band grid: offsets in the upper half are negative and keep their
    distance to the end of the grid; multiplicities scale with the band size (a partially
    walked group keeps its fraction). At K = 3N the reference's kept generator sets at 256^2
    and 1024^2 agree up to near-tie order (tests/test_varying.py)."""
    old = make_layout(gl.dims, gl.J)
    new = make_layout(new_dims, gl.J)
    nb = len(old.bands)
    gi = np.empty_like(gl.gen_index)
    cnt = np.empty_like(gl.counts)
    for k in range(gl.blocks.size):
        b = int(gl.blocks[k])
        bi_o, bo_o = old.bands[b % nb], old.bands[b // nb]
        bi_n, bo_n = new.bands[b % nb], new.bands[b // nb]
        in_finer = bi_o.level <= bo_o.level
        gs_o = bi_o.shape if in_finer else bo_o.shape
        gs_n = bi_n.shape if in_finer else bo_n.shape
        small_o = bo_o if in_finer else bi_o
        small_n = bo_n if in_finer else bi_n
        rem = int(gl.gen_index[k])
        v = []
        for s in reversed(gs_o):
            v.append(rem % s)
            rem //= s
        v = v[::-1]
        v2 = [vk if vk < so // 2 else vk + (sn - so) for vk, so, sn in zip(v, gs_o, gs_n)]
        flat = 0
        for vk, sn in zip(v2, gs_n):
            flat = flat * sn + vk
        gi[k] = flat
        c = int(gl.counts[k])
        cnt[k] = small_n.count() if c == small_o.count() else int(round(c * small_n.count() / small_o.count()))
    return GeneratorList(tuple(int(d) for d in new_dims), gl.J, gl.family, gl.order, gl.blocks.copy(), gi, cnt,
                         gl.values.copy())


def json_dims(z):
    import json
    return json.loads(bytes(z["meta_json"]).decode())["dims"]


def theta_varying(ladder: SigmaLadder, sigma_first_row: float = 2.5, sigma_last_row: float = 7.5) -> SparseOperator:
    """Spatially varying Theta_K (BASELINE C3/C4): column-wise interpolation across a sigma
    ladder of stationary operators (wbx_theta_varying; no reference implementation)."""
    g0 = ladder.levels[0]
    dims = np.array(g0.dims, dtype=np.uint64)
    ngens = np.array([g.blocks.size for g in ladder.levels], dtype=np.uint64)
    cat = lambda attr, dt: np.ascontiguousarray(np.concatenate([getattr(g, attr) for g in ladder.levels]).astype(dt))
    blocks, gidx = cat("blocks", np.uint32), cat("gen_index", np.uint32)
    counts, vals = cat("counts", np.uint64), cat("values", np.float64)
    sig = np.ascontiguousarray(ladder.sigmas, dtype=np.float64)
    nnz = C.c_uint64()
    ro_p, ci_p, va_p = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint32)(), C.POINTER(C.c_double)()
    _check(lib.wbx_theta_varying(len(g0.dims), _u64ptr(dims), g0.J, sig.size, _dptr(sig), _u64ptr(ngens),
                                 _u32ptr(blocks), _u32ptr(gidx), _u64ptr(counts), _dptr(vals),
                                 float(sigma_first_row), float(sigma_last_row), C.byref(nnz), C.byref(ro_p),
                                 C.byref(ci_p), C.byref(va_p)))
    layout = make_layout(g0.dims, g0.J)
    n = layout.total()
    try:
        ro = np.ctypeslib.as_array(ro_p, shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(ci_p, shape=(max(nnz.value, 1),))[: nnz.value].copy()
        va = np.ctypeslib.as_array(va_p, shape=(max(nnz.value, 1),))[: nnz.value].copy()
    finally:
        for p in (ro_p, ci_p, va_p):
            lib.wbx_free(C.cast(p, C.c_void_p))
    return SparseOperator(n, ro, ci, va, layout, g0.family, g0.order)


# ----------------------------------------------------------------------------- weights
@dataclass
class WeightVector:
    sigma: np.ndarray


def uniform_weights(layout: SubbandLayout) -> WeightVector:
    return WeightVector(np.ones(layout.total()))


def dyadic_weights(layout: SubbandLayout) -> WeightVector:
    """sigma = 2^(t-J) of the coefficient's band (theta.cpp:153-165)."""
    s = np.empty(layout.total())
    for b in layout.bands:
        s[b.offset:b.offset + b.count()] = 2.0 ** (b.level - layout.J)
    return WeightVector(s)


def scale_weights(layout: SubbandLayout) -> np.ndarray:
    """w = level t on detail bands, J on the approximation (solver.cpp:33-42)."""
    d = np.array(layout.dims, dtype=np.uint64)
    w = np.empty(layout.total())
    _check(lib.wbx_scale_weights(len(layout.dims), _u64ptr(d), layout.J, _dptr(w)))
    return w


# ----------------------------------------------------------------------------- preconditioners
class PrecondKind(enum.IntEnum):
    Identity = 0
    Jacobi = 1
    Spai = 2


@dataclass
class DiagonalPreconditioner:  # precond.hpp:11-14
    p: np.ndarray
    kind: PrecondKind = PrecondKind.Identity


def identity_precond(n: int) -> DiagonalPreconditioner:
    return DiagonalPreconditioner(np.ones(n), PrecondKind.Identity)


@dataclass
class GramDiagonals:
    diagM: np.ndarray
    diagM2: np.ndarray


def gram_diagonals(op: SparseOperator, nnz_cap_factor: int = 50, ctx=None) -> GramDiagonals:
    """precond.cpp:16-67 (exact fp64, same accumulation order)."""
    ctx = _ctx_of(op, ctx)
    m = np.empty(op.n)
    m2 = np.empty(op.n)
    _check(lib.wbx_gram_diagonals(ctx.handle, op.device(ctx), nnz_cap_factor, _dptr(m), _dptr(m2)))
    return GramDiagonals(m, m2)


def spai(op: SparseOperator, ctx=None) -> DiagonalPreconditioner:
    ctx = _ctx_of(op, ctx)
    p = np.empty(op.n)
    _check(lib.wbx_spai(ctx.handle, op.device(ctx), _dptr(p)))
    return DiagonalPreconditioner(p, PrecondKind.Spai)


def jacobi(op: SparseOperator, eps: float, ctx=None) -> DiagonalPreconditioner:
    if eps <= 0.0:
        raise BadEpsilon("jacobi: epsilon must be positive")
    ctx = _ctx_of(op, ctx)
    p = np.empty(op.n)
    _check(lib.wbx_jacobi(ctx.handle, op.device(ctx), float(eps), _dptr(p)))
    return DiagonalPreconditioner(p, PrecondKind.Jacobi)


# ----------------------------------------------------------------------------- solver
class SparseThetaOp:
    """ThetaOp over a SparseOperator (solver.hpp:25-38)."""

    def __init__(self, op: SparseOperator, ctx: Optional[Context] = None):
        self._op = op
        self._ctx = ctx

    def apply(self, x) -> np.ndarray:
        return spmv(self._op, x, self._ctx)

    def apply_adjoint(self, x) -> np.ndarray:
        return spmv_t(self._op, x, self._ctx)

    def dim(self) -> int:
        return self._op.n

    def ops_per_pixel(self) -> float:
        return ops_per_pixel(self._op)

    def sparse(self) -> SparseOperator:
        return self._op


class ExactThetaOp:
    """ThetaOp of the exact FFT operator (solver.hpp:41-52, solver.cpp:21-29) on the device:
    Theta x = analyze(convolve(synthesize(x), psf)); bitwise the reference's (oracle FFT
    arithmetic). psf: the kernel image (e.g. gaussian_psf_kernel)."""

    def __init__(self, psf_kernel, basis: WaveletBasis, ctx: Optional[Context] = None):
        self._ctx = ctx or default_context()
        self.basis = basis
        self.n = basis.layout.total()
        k = _f64(np.asarray(psf_kernel, dtype=np.float64).ravel(), self.n, "psf kernel")
        h = C.c_void_p()
        _check(lib.wbx_exact_op_create(self._ctx.handle, basis.device(self._ctx), _dptr(k), C.byref(h)))
        self.handle = h

    def _apply(self, x, adjoint: int) -> np.ndarray:
        xv = _f64(x, self.n)
        y = np.empty(self.n)
        _check(lib.wbx_exact_apply(self.handle, adjoint, _dptr(xv), _dptr(y)))
        return y

    def apply(self, x) -> np.ndarray:
        return self._apply(x, 0)

    def apply_adjoint(self, x) -> np.ndarray:
        return self._apply(x, 1)

    def dim(self) -> int:
        return self.n

    def __del__(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        if getattr(self, "handle", None):
            lib.wbx_exact_op_destroy(self.handle)
            self.handle = None


@dataclass
class DeblurProblem:  # solver.hpp:55-61
    op: SparseThetaOp = None
    x0: np.ndarray = None
    weights: np.ndarray = None
    lambda_: float = 1e-4


@dataclass
class SolverConfig:  # solver.hpp:66-74 (+ device knobs)
    max_iters: int = 500
    rel_energy_tol: float = 1e-3
    step_safety: float = 1.01
    track_support: bool = False
    ref_energy: float = math.nan
    zero_momentum: bool = False
    track_energy: bool = True   # the reference always records energies
    precision: int = N.WBX_FP32
    tau: float = 0.0            # > 0: given step (skips estimate_step)

    def to_c(self) -> N.wbx_solver_cfg:
        c = N.wbx_solver_cfg()
        c.max_iters = int(self.max_iters)
        c.rel_energy_tol = float(self.rel_energy_tol)
        c.step_safety = float(self.step_safety)
        c.ref_energy = float(self.ref_energy)
        c.zero_momentum = int(bool(self.zero_momentum))
        c.track_support = int(bool(self.track_support))
        c.track_energy = int(bool(self.track_energy))
        c.precision = int(self.precision)
        c.tau = float(self.tau or 0.0)
        return c


@dataclass
class SolveReport:  # solver.hpp:76-84
    x_final: np.ndarray = None
    energies: list = field(default_factory=list)
    iters_used: int = 0
    support_sizes: list = field(default_factory=list)
    wall_time_s: float = 0.0
    ops_per_pixel_per_iter: float = 0.0
    initial_energy: float = 0.0
    tau: float = 0.0
    tau_iters: int = 0


def energy(x, problem: DeblurProblem, ctx=None) -> float:
    """½‖Θx − x0‖² + λ Σ w|x| (solver.cpp:44-55)."""
    if isinstance(problem.op, ExactThetaOp):
        r = problem.op.apply(x) - _f64(problem.x0)
        return 0.5 * float(np.dot(r, r)) + problem.lambda_ * float(np.dot(_f64(problem.weights), np.abs(_f64(x))))
    op = problem.op.sparse()
    xv = _f64(x)
    if xv.size != len(problem.x0):
        raise ShapeMismatch("energy: vector length mismatch")
    ctx = _ctx_of(op, ctx)
    e = C.c_double()
    _check(lib.wbx_energy(ctx.handle, op.device(ctx), _dptr(xv), _dptr(_f64(problem.x0)),
                          _dptr(_f64(problem.weights)), float(problem.lambda_), C.byref(e)))
    return e.value


def prox_weighted_l1_P(z0, tau: float, weights, lambda_: float, P: DiagonalPreconditioner,
                       ctx=None) -> np.ndarray:
    """z = sign(z0) max(|z0| − τλw/p, 0) (solver.cpp:57-67), on the device."""
    z0v = _f64(z0)
    n = z0v.size
    w = _f64(weights, n, "weights")
    p = _f64(P.p, n, "preconditioner")
    ctx = ctx or default_context()
    z = np.empty(n)
    _check(lib.wbx_prox_l1w(ctx.handle, n, _dptr(z0v), float(tau), _dptr(w), float(lambda_), _dptr(p),
                            _dptr(z)))
    return z


def estimate_step(op: SparseThetaOp, P: DiagonalPreconditioner, step_safety: float = 1.0,
                  ctx=None, return_iters: bool = False):
    """τ = 1/(step_safety ‖P^-½ΘᵀΘP^-½‖) by the reference's power iteration (solver.cpp:69-99)."""
    if isinstance(op, ExactThetaOp):
        p = _f64(P.p, op.n, "preconditioner")
        tau, it = C.c_double(), C.c_uint32()
        _check(lib.wbx_estimate_step_exact(op.handle, _dptr(p), float(step_safety), C.byref(tau), C.byref(it)))
        return (tau.value, it.value) if return_iters else tau.value
    sp = op.sparse()
    ctx = _ctx_of(sp, ctx)
    p = _f64(P.p, sp.n, "preconditioner")
    tau = C.c_double()
    it = C.c_uint32()
    _check(lib.wbx_estimate_step(ctx.handle, sp.device(ctx), _dptr(p), float(step_safety), C.byref(tau),
                                 C.byref(it)))
    return (tau.value, it.value) if return_iters else tau.value


def _run_pgd(problem: DeblurProblem, P: DiagonalPreconditioner, config: SolverConfig, accelerate: int,
             ctx=None) -> SolveReport:
    if isinstance(problem.op, ExactThetaOp):
        return _run_pgd_exact(problem, P, config, accelerate)
    sp = problem.op.sparse()
    n = sp.n
    x0 = _f64(problem.x0)
    w = _f64(problem.weights)
    p = _f64(P.p)
    if x0.size != n or w.size != n or p.size != n:
        raise ShapeMismatch("solver: inconsistent problem dimensions")
    ctx = _ctx_of(sp, ctx)
    cfg = config.to_c()
    K = int(config.max_iters)
    energies = np.zeros(max(K, 1))
    supports = np.zeros(max(K, 1), dtype=np.uint64)
    rep = N.wbx_report()
    rep.energies = _dptr(energies)
    rep.support_sizes = _u64ptr(supports)
    xf = np.empty(n)
    _check(lib.wbx_pgd(ctx.handle, sp.device(ctx), _dptr(x0), _dptr(w), float(problem.lambda_), _dptr(p),
                       C.byref(cfg), accelerate, _dptr(xf), C.byref(rep)))
    used = int(rep.iters_used)
    track = config.track_energy or config.track_support or math.isfinite(config.ref_energy)
    return SolveReport(
        x_final=xf,
        energies=list(energies[:used]) if track else [],
        iters_used=used,
        support_sizes=[int(s) for s in supports[:used]] if (track and config.track_support) else [],
        wall_time_s=rep.wall_time_s,
        ops_per_pixel_per_iter=rep.ops_per_pixel_per_iter,
        initial_energy=rep.initial_energy,
        tau=rep.tau,
        tau_iters=int(rep.tau_iters))


def _run_pgd_exact(problem: DeblurProblem, P: DiagonalPreconditioner, config: SolverConfig,
                   accelerate: int) -> SolveReport:
    """run_pgd over the exact FFT operator (fp64, the reference's expressions)."""
    op = problem.op
    n = op.n
    x0, w, p = _f64(problem.x0), _f64(problem.weights), _f64(P.p)
    if x0.size != n or w.size != n or p.size != n:
        raise ShapeMismatch("solver: inconsistent problem dimensions")
    cfg = config.to_c()
    K = int(config.max_iters)
    energies = np.zeros(max(K, 1))
    supports = np.zeros(max(K, 1), dtype=np.uint64)
    rep = N.wbx_report()
    rep.energies = _dptr(energies)
    rep.support_sizes = _u64ptr(supports)
    xf = np.empty(n)
    _check(lib.wbx_pgd_exact(op.handle, _dptr(x0), _dptr(w), float(problem.lambda_), _dptr(p), C.byref(cfg),
                             accelerate, _dptr(xf), C.byref(rep)))
    used = int(rep.iters_used)
    track = config.track_energy or math.isfinite(config.ref_energy)
    return SolveReport(x_final=xf, energies=list(energies[:used]) if track else [], iters_used=used,
                       support_sizes=[int(v) for v in supports[:used]] if config.track_support else [],
                       wall_time_s=rep.wall_time_s, ops_per_pixel_per_iter=rep.ops_per_pixel_per_iter,
                       initial_energy=rep.initial_energy, tau=rep.tau, tau_iters=int(rep.tau_iters))


def ista(problem: DeblurProblem, P: DiagonalPreconditioner, config: SolverConfig, ctx=None) -> SolveReport:
    """solver.cpp:161-164."""
    return _run_pgd(problem, P, config, 0, ctx)


def fista(problem: DeblurProblem, P: DiagonalPreconditioner, config: SolverConfig, ctx=None) -> SolveReport:
    """Preconditioned accelerated proximal gradient, momentum (k−1)/(k+2) (solver.cpp:166-169)."""
    return _run_pgd(problem, P, config, 1, ctx)


# ----------------------------------------------------------------------------- prepared deblur
class Deblurrer:
    """The deblur unit of the reference CLI (waveblur.cpp:286-297) with the operator,
    preconditioner, weights and λ bound once: u0 → analyze → [estimate_step] → FISTA →
    synthesize (→ clamp). `deblur` takes host arrays; `deblur_dev` device pointers."""

    def __init__(self, op: SparseOperator, basis: WaveletBasis, P: DiagonalPreconditioner, weights,
                 lambda_: float, config: SolverConfig, ctx: Optional[Context] = None, batch: int = 1):
        self.ctx = ctx or op._ctx or default_context()
        self.op, self.basis, self.config = op, basis, config
        self.n = op.n
        self.batch = int(batch)
        p = _f64(P.p, op.n, "preconditioner")
        w = _f64(weights, op.n, "weights")
        cfg = config.to_c()
        h = C.c_void_p()
        _check(lib.wbx_solver_create_batch(self.ctx.handle, op.device(self.ctx), basis.device(self.ctx), _dptr(p),
                                           _dptr(w), float(lambda_), C.byref(cfg), self.batch, C.byref(h)))
        self.handle = h

    def deblur(self, u0: np.ndarray, clamp: bool = True, out: Optional[np.ndarray] = None):
        """u0: one image (batch 1) or `batch` images stacked on the first axis."""
        u = _f64(u0, self.n * self.batch, "u0")
        res = out if out is not None else np.empty(self.n * self.batch)
        rep = N.wbx_report()
        _check(lib.wbx_deblur(self.handle, _dptr(u), res.ctypes.data_as(C.POINTER(C.c_double)), int(clamp),
                              C.byref(rep)))
        shape = tuple(self.basis.layout.dims) if self.batch == 1 else (self.batch,) + tuple(self.basis.layout.dims)
        return res.reshape(shape), rep

    def deblur_dev(self, u0_ptr: int, u_ptr: int, clamp: bool = True) -> None:
        _check(lib.wbx_deblur_dev(self.handle, C.c_void_p(u0_ptr), C.c_void_p(u_ptr), int(clamp)))

    def last_stats(self):
        launches = C.c_uint64()
        ms = C.c_float()
        _check(lib.wbx_solver_last_stats(self.handle, C.byref(launches), C.byref(ms)))
        return int(launches.value), float(ms.value)

    def phase_ms(self):
        """(estimate_step ms, iteration-kernel ms) of the last solve (device events)."""
        t, i = C.c_float(), C.c_float()
        _check(lib.wbx_solver_phase_ms(self.handle, C.byref(t), C.byref(i)))
        return float(t.value), float(i.value)

    def kernels(self):
        """(step-estimate kernel, iteration kernel) names of the engine this solver runs."""
        buf = C.create_string_buffer(256)
        _check(lib.wbx_solver_kernels(self.handle, buf, 256))
        return tuple(buf.value.decode().split(" ", 1))

    def tau_stats(self):
        """(tau, the reference's power-iteration count, operator product pairs spent) of the
        last solve (Lanczos steps on the fp32 hot path)."""
        t, it, pp = C.c_double(), C.c_uint32(), C.c_uint32()
        _check(lib.wbx_solver_tau_stats(self.handle, C.byref(t), C.byref(it), C.byref(pp)))
        return float(t.value), int(it.value), int(pp.value)

    def __del__(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        if getattr(self, "handle", None):
            lib.wbx_solver_destroy(self.handle)
            self.handle = None
