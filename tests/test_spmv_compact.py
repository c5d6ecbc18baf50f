"""The SELL SpMV kernel alone in the compacted spaces (wbx_spmv_compact_dev, the kernel
tools/spmv_roofline.py measures) against the full-vector entry point wbx_spmv_dev, whose
fp64 form is bitwise the reference's spmv (theta.cpp:300-311, test_gpu_parity.py):
y_compact == y_full[R] bitwise, fp64 and fp32, forward and adjoint."""
import ctypes as C

import numpy as np
import pytest

from paper_1512_08401_b200 import _native as N
from paper_1512_08401_b200 import waveblur as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["s128_1d_sym6", "s64_sym6_spai", "c1_db4_256", "c2_db4_1024"])
def test_compact_spmv_equals_full(golden, name):
    import torch
    g = golden(name)
    op = g.operator()
    ctx = W.default_context()
    h = op.device(ctx)
    rp = np.asarray(op.row_offsets, dtype=np.uint64)
    # compacted spaces: nonempty rows / columns by descending length, stable on index
    # (op_build.cu)
    rlen = np.diff(rp).astype(np.int64)
    clen = np.bincount(np.asarray(op.col_indices, dtype=np.int64), minlength=op.n)
    R = np.nonzero(rlen)[0]
    R = R[np.argsort(-rlen[R], kind="stable")]
    Cc = np.nonzero(clen)[0]
    Cc = Cc[np.argsort(-clen[Cc], kind="stable")]
    inf = op.info(ctx)
    assert (inf.nonempty_rows, inf.nonempty_cols) == (R.size, Cc.size)
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(7)
    for prec, dt in ((N.WBX_FP64, torch.float64), (N.WBX_FP32, torch.float32)):
        for transpose in (False, True):
            src, dst = (R, Cc) if transpose else (Cc, R)
            xf = torch.from_numpy(rng.standard_normal(op.n)).to(dev, dt)
            yf = torch.empty_like(xf)
            xc = xf[torch.from_numpy(src.astype(np.int64)).to(dev)].contiguous()
            yc = torch.empty(dst.size, dtype=dt, device=dev)
            torch.cuda.synchronize()
            W._check(N.lib.wbx_spmv_dev(ctx.handle, h, int(transpose), prec, C.c_void_p(xf.data_ptr()),
                                        C.c_void_p(yf.data_ptr())))
            W._check(N.lib.wbx_spmv_compact_dev(ctx.handle, h, int(transpose), prec,
                                                C.c_void_p(xc.data_ptr()), C.c_void_p(yc.data_ptr())))
            ctx.synchronize()
            full = yf.cpu().numpy()
            assert np.array_equal(yc.cpu().numpy(), full[dst]), (name, prec, transpose)
            mask = np.ones(op.n, bool)
            mask[dst] = False
            assert not full[mask].any()
