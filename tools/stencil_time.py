"""Stencil SpMV (circulant-compressed Theta_K, reads only x and y) vs the CSR-derived sliced-ELL
SpMV (wbx_spmv_dev) at C2, fp32 and fp64, forward and adjoint: device time per SpMV (CUDA
events on the context stream, L2 warm) and the bytes each moves."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1512_08401_b200 import _native as N  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

z = np.load(bench.GOLDEN)
gl = W.GeneratorList(bench.DIMS, 4, W.FilterFamily.Daubechies, 4, z["gen_block"].astype(np.uint32),
                     z["gen_index"].astype(np.uint32), z["gen_count"].astype(np.uint64), z["gen_value"])
op = W.theta_from_generators(gl)
ctx = W.default_context()
st = W.StencilOperator(gl, ctx)
dev = torch.device("cuda", 0)
stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
n, nnz = op.n, op.nnz()
res = {"n": n, "nnz": nnz, "records": int(gl.blocks.size)}
for prec, dt in ((N.WBX_FP32, torch.float32), (N.WBX_FP64, torch.float64)):
    with torch.cuda.stream(stream):
        x = torch.randn(n, dtype=dt, device=dev)
        y = torch.empty_like(x)
    torch.cuda.synchronize()
    for name, fn in (("stencil", lambda t: st.spmv_dev(x.data_ptr(), y.data_ptr(), t, prec)),
                     ("sell", lambda t: W._check(N.lib.wbx_spmv_dev(ctx.handle, op.device(ctx), int(t), prec,
                                                                   C.c_void_p(x.data_ptr()),
                                                                   C.c_void_p(y.data_ptr()))))):
        for t in (False, True):
            for _ in range(3):
                fn(t)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                a.record(stream)
            for _ in range(20):
                fn(t)
            with torch.cuda.stream(stream):
                b.record(stream)
            b.synchronize()
            us = 1e3 * a.elapsed_time(b) / 20
            res[f"{name}_{'adj' if t else 'fwd'}_fp{64 if prec == N.WBX_FP64 else 32}_us"] = round(us, 2)
w = 4
res["stencil_bytes_fp32"] = 2 * w * n
res["csr_algorithmic_bytes_fp32 (8nnz+8n)"] = 8 * nnz + 8 * n
print(json.dumps(res))
