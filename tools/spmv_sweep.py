"""Sweep of the standalone fp32 SpMV kernels (wbx_diag_spmv_compact_mode) and the row
kernel's L2 prefetch distance on the 4096^2 operator of tools/spmv_roofline.py (L2 flushed
before every call, CUDA events, median of REPS). Prints one JSON line per configuration.
  python tools/spmv_sweep.py [SIDE] [REPS] [modes] [pf_mib,...]"""
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

MODES = {"reg": 0, "tma1": 1, "tma2": 2, "tma3": 3, "half": 4, "quarter": 5, "row2": 6, "row": 7, "row8": 8}
side = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["quarter", "row2", "row", "row8"]
pfs = [float(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0, 4, 16, 64]
z = np.load(ROOT / "tests" / "golden" / "c2_db4_1024.npz")
gl = W.GeneratorList((1024, 1024), 4, W.FilterFamily.Daubechies, 4, z["gen_block"].astype(np.uint32),
                     z["gen_index"].astype(np.uint32), z["gen_count"].astype(np.uint64), z["gen_value"])
if side != 1024:
    gl = W.rescale_generators(gl, (side, side))
op = W.theta_from_generators(gl)
ctx = W.default_context()
h = op.device(ctx)
inf = op.info(ctx)
nnz, nR, nC = int(inf.nnz), int(inf.nonempty_rows), int(inf.nonempty_cols)
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6545.3
dev = torch.device("cuda", 0)
stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
with torch.cuda.stream(stream):
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    xR = torch.randn(max(nR, 1), device=dev)
    xC = torch.randn(max(nC, 1), device=dev)
    yR = torch.empty(max(nR, 1), device=dev)
    yC = torch.empty(max(nC, 1), device=dev)
torch.cuda.synchronize()
b = 8 * nnz + 4 * (nR + nC)
for m in modes:
    for pf in (pfs if m.startswith("row") else [None]):
        if pf is not None:
            N.lib.wbx_diag_set_spmv_pf(int(pf * (1 << 20)))
        for t in (0, 1):
            x, y = (xR, yC) if t else (xC, yR)
            def call():
                W._check(N.lib.wbx_diag_spmv_compact_mode(ctx.handle, h, t, MODES[m], C.c_void_p(x.data_ptr()),
                                                          C.c_void_p(y.data_ptr())))
            for _ in range(3):
                call()
            ms = []
            for _ in range(reps):
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    flush.fill_(1)
                    a.record(stream)
                call()
                with torch.cuda.stream(stream):
                    e.record(stream)
                e.synchronize()
                ms.append(a.elapsed_time(e))
            med = statistics.median(ms)
            print(json.dumps({"mode": m, "pf_mib": pf, "side": "adj" if t else "fwd", "us": round(1e3 * med, 2),
                              "gbs": round(b / med / 1e6, 1), "frac": round(b / med / 1e6 / peak, 4)}), flush=True)
N.lib.wbx_diag_set_spmv_pf(-1)
