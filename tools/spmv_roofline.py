"""Theta x SpMV against the HBM roofline (the second half of BASELINE.json's metric).

Operator: the reference's C2 thresholded operator (tests/golden/c2_db4_1024.npz, K = 3N)
carried to an SIDE x SIDE grid by rescale_generators (default 4096^2: nnz ~ 50 M, 400 MB of
fp32 value + u32 index stream, > 126 MB L2, so the SpMV streams from HBM). The L2 is also
flushed (512 MiB write) before every timed call.

Timed with CUDA events on the context stream, per call, median of REPS:
  * sell kernel alone (wbx_spmv_compact_dev), forward (Theta) and adjoint (Theta^T), fp32;
  * the full-vector entry point wbx_spmv_dev (memset y + gather x + sell + scatter y).
Algorithmic bytes: 8*nnz + 4*n + 4*n for the full-vector SpMV; for the kernel
alone 8*nnz + 4*|C| + 4*|R| (its compacted input and output).

  python tools/spmv_roofline.py [SIDE] [REPS]
"""
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_1512_08401_b200 import _native as N  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402


def measure(side: int = 4096, reps: int = 20) -> dict:
    """Time the SELL kernel and the full-vector SpMV at SIDE^2 (see module docstring)."""
    dims = (side, side)
    z = np.load(ROOT / "tests" / "golden" / "c2_db4_1024.npz")
    gl = W.GeneratorList((1024, 1024), 4, W.FilterFamily.Daubechies, 4, z["gen_block"].astype(np.uint32),
                         z["gen_index"].astype(np.uint32), z["gen_count"].astype(np.uint64), z["gen_value"])
    if side != 1024:
        gl = W.rescale_generators(gl, dims)
    op = W.theta_from_generators(gl)
    ctx = W.default_context()
    h = op.device(ctx)
    inf = op.info(ctx)
    n, nnz = int(inf.n), int(inf.nnz)
    nR, nC = int(inf.nonempty_rows), int(inf.nonempty_cols)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 7672.0
    dev = torch.device("cuda", 0)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    with torch.cuda.stream(stream):
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        xf = torch.randn(n, device=dev)
        yf = torch.empty(n, device=dev)
        xR = torch.randn(max(nR, 1), device=dev)
        xC = torch.randn(max(nC, 1), device=dev)
        yR = torch.empty(max(nR, 1), device=dev)
        yC = torch.empty(max(nC, 1), device=dev)
    torch.cuda.synchronize()

    def compact(t):
        x, y = (xR, yC) if t else (xC, yR)
        W._check(N.lib.wbx_spmv_compact_dev(ctx.handle, h, int(t), N.WBX_FP32, C.c_void_p(x.data_ptr()),
                                            C.c_void_p(y.data_ptr())))

    def full(t):
        W._check(N.lib.wbx_spmv_dev(ctx.handle, h, int(t), N.WBX_FP32, C.c_void_p(xf.data_ptr()),
                                    C.c_void_p(yf.data_ptr())))

    def timed(fn, t):
        for _ in range(3):
            fn(t)
        ms = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                flush.fill_(1)
                a.record(stream)
            fn(t)
            with torch.cuda.stream(stream):
                b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        return statistics.median(ms)

    res = {"grid": list(dims), "n": n, "nnz": nnz, "nonempty_rows": nR, "nonempty_cols": nC,
           "operator_stream_bytes_model": 8 * nnz, "l2": "flushed (512 MiB write) before every call",
           "peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    for t, name in ((False, "fwd"), (True, "adj")):
        ms = timed(compact, t)
        b = 8 * nnz + 4 * (nR + nC)
        res[f"sell_{name}"] = {"us": round(1e3 * ms, 2), "algorithmic_bytes": b,
                               "gbs": round(b / ms / 1e6, 1), "frac": round(b / ms / 1e6 / peak, 3)}
        ms = timed(full, t)
        b = 8 * nnz + 8 * n
        res[f"full_{name}"] = {"us": round(1e3 * ms, 2), "algorithmic_bytes": b,
                               "gbs": round(b / ms / 1e6, 1), "frac": round(b / ms / 1e6 / peak, 3),
                               "launches": "memset + gather + sell + scatter"}
    return res


if __name__ == "__main__":
    print(json.dumps(measure(int(sys.argv[1]) if len(sys.argv) > 1 else 4096,
                             int(sys.argv[2]) if len(sys.argv) > 2 else 20)))
