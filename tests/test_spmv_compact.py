"""The SELL SpMV kernels alone in the compacted spaces (wbx_spmv_compact_dev, the kernel
tools/spmv_roofline.py measures).

* against the full-vector entry point wbx_spmv_dev (fp64 form bitwise the reference's spmv,
  theta.cpp:300-311; test_gpu_parity.py): y_compact == y_full[R] bitwise, fp64 and fp32;
* every fp32 kernel variant, selected explicitly (wbx_diag_spmv_compact_mode; WBX_SPMV is read
  once per process), against the oracle's fp64 spmv (oracle/wbx_oracle.c, pinned bitwise to the
  reference): |y - y_ref| <= 1e-6 * max|y_ref| (fp32 values and vector entries, fp32 sums);
* variants sharing a summation order are bitwise equal: the segmented kernels (reg, tma1-3,
  half, quarter) among themselves, the row-per-lane kernels (row, row2, row8) among themselves."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_08401_b200 import _native as N
from paper_1512_08401_b200 import waveblur as W

pytestmark = pytest.mark.gpu

MODES = {"reg": 0, "tma1": 1, "tma2": 2, "tma3": 3, "half": 4, "quarter": 5, "row2": 6, "row": 7, "row8": 8}
SEGMENTED = ("reg", "tma1", "tma2", "tma3", "half", "quarter")
ROW = ("row", "row2", "row8")


def compacted_spaces(op):
    """Nonempty rows / columns by descending length, stable on index (op_build.cu)."""
    rp = np.asarray(op.row_offsets, dtype=np.uint64)
    rlen = np.diff(rp).astype(np.int64)
    clen = np.bincount(np.asarray(op.col_indices, dtype=np.int64), minlength=op.n)
    R = np.nonzero(rlen)[0]
    R = R[np.argsort(-rlen[R], kind="stable")]
    Cc = np.nonzero(clen)[0]
    Cc = Cc[np.argsort(-clen[Cc], kind="stable")]
    return R, Cc


@pytest.mark.parametrize("name", ["s128_1d_sym6", "s64_sym6_spai", "c1_db4_256", "c2_db4_1024"])
def test_compact_spmv_equals_full(golden, name):
    import torch
    g = golden(name)
    op = g.operator()
    ctx = W.default_context()
    h = op.device(ctx)
    R, Cc = compacted_spaces(op)
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


def run_mode(ctx, h, transpose, mode, xc, ny):
    import torch
    yc = torch.full((max(ny, 1),), float("nan"), dtype=torch.float32, device=xc.device)
    torch.cuda.synchronize()
    W._check(N.lib.wbx_diag_spmv_compact_mode(ctx.handle, h, int(transpose), mode, C.c_void_p(xc.data_ptr()),
                                              C.c_void_p(yc.data_ptr())))
    ctx.synchronize()
    return yc.cpu().numpy()[:ny]


@pytest.mark.parametrize("name", ["s128_1d_sym6", "s64_sym6_spai", "c1_db4_256", "c2_db4_1024"])
def test_fp32_kernels_vs_oracle_and_each_other(golden, name):
    import torch
    g = golden(name)
    op = g.operator()
    ctx = W.default_context()
    h = op.device(ctx)
    R, Cc = compacted_spaces(op)
    A = O.Csr.of(op)
    AT = A.transpose()
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(11)
    for transpose in (False, True):
        src, dst = (R, Cc) if transpose else (Cc, R)
        x = rng.standard_normal(op.n).astype(np.float32).astype(np.float64)  # fp32-exact input
        ref = O.spmv(AT if transpose else A, x)[dst]
        xc = torch.from_numpy(x[src].astype(np.float32)).to(dev)
        out = {m: run_mode(ctx, h, transpose, k, xc, dst.size) for m, k in MODES.items()}
        scale = max(np.abs(ref).max(), 1e-300)
        for m, y in out.items():
            assert np.all(np.isfinite(y)), (name, m, transpose)
            err = np.abs(y.astype(np.float64) - ref).max() / scale
            assert err <= 1e-6, (name, m, transpose, err)
        for m in SEGMENTED[1:]:
            assert np.array_equal(out[m], out[SEGMENTED[0]]), (name, m, transpose)
        assert np.array_equal(out["row2"], out["row"]) and np.array_equal(out["row8"], out["row"]), (name, transpose)


def test_fp32_row_kernel_at_4096_vs_oracle():
    """The operator tools/spmv_roofline.py measures (C2's Theta_K carried to 4096^2, 50 M
    nonzeros, HBM-streamed): the default row kernel, forward and adjoint, against the
    oracle's fp64 spmv on a sample of rows (1e-6 of max|y|) and bitwise against row2 / row8."""
    import torch
    from pathlib import Path
    z = np.load(Path(__file__).resolve().parent / "golden" / "c2_db4_1024.npz")
    gl = W.GeneratorList((1024, 1024), 4, W.FilterFamily.Daubechies, 4, z["gen_block"].astype(np.uint32),
                         z["gen_index"].astype(np.uint32), z["gen_count"].astype(np.uint64), z["gen_value"])
    op = W.theta_from_generators(W.rescale_generators(gl, (4096, 4096)))
    ctx = W.default_context()
    h = op.device(ctx)
    R, Cc = compacted_spaces(op)
    rp = np.asarray(op.row_offsets, dtype=np.int64)
    cols = np.asarray(op.col_indices, dtype=np.int64)
    vals = np.asarray(op.values)
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    x = rng.standard_normal(op.n).astype(np.float32).astype(np.float64)
    xc = torch.from_numpy(x[Cc].astype(np.float32)).to(dev)
    y = run_mode(ctx, h, False, MODES["row"], xc, R.size)
    assert np.array_equal(y, run_mode(ctx, h, False, MODES["row2"], xc, R.size))
    assert np.array_equal(y, run_mode(ctx, h, False, MODES["row8"], xc, R.size))
    sample = rng.choice(R.size, 20000, replace=False)
    ref = np.array([vals[rp[r]:rp[r + 1]] @ x[cols[rp[r]:rp[r + 1]]] for r in R[sample]])
    assert np.abs(y[sample] - ref).max() <= 1e-6 * np.abs(ref).max()
    # adjoint: y_T[c] = sum_r Theta[r, c] x[r] over the compacted column space
    xr = rng.standard_normal(op.n).astype(np.float32).astype(np.float64)
    xrc = torch.from_numpy(xr[R].astype(np.float32)).to(dev)
    yt = run_mode(ctx, h, True, MODES["row"], xrc, Cc.size)
    full = np.zeros(op.n)
    np.add.at(full, cols, vals * np.repeat(xr, np.diff(rp)))
    reft = full[Cc]
    assert np.abs(yt - reft).max() <= 1e-6 * np.abs(reft).max()
