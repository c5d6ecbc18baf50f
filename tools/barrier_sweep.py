"""C2 deblur time vs the counter barrier's number of arrival groups (WBX_BARRIER_GROUPS): one
Deblurrer per setting (the setting is captured with its graphs), L2 flushed between steps,
CUDA events, median of STEPS.
  python tools/barrier_sweep.py [groups,...] [steps]"""
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

groups = [int(g) for g in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 4, 8, 16]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
op, basis, u0 = bench.make_inputs()
ctx = W.Context(0)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
dev = torch.device("cuda", 0)
stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
with torch.cuda.stream(stream):
    u = torch.from_numpy(u0.ravel().copy()).to(dev)
    out = torch.empty_like(u)
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
ref = None
for g in groups:
    os.environ["WBX_BARRIER_GROUPS"] = str(g)
    d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False), ctx)
    for _ in range(3):
        d.deblur_dev(u.data_ptr(), out.data_ptr())
    ms, ph = [], []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.zero_()
            a.record(stream)
        d.deblur_dev(u.data_ptr(), out.data_ptr())
        with torch.cuda.stream(stream):
            b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
        ph.append(d.phase_ms())
    img = out.cpu().numpy()
    same = None if ref is None else bool((img == ref).all())
    ref = img if ref is None else ref
    print(json.dumps({"groups": g, "ms": round(statistics.median(ms), 4),
                      "tau_ms": round(statistics.median(p[0] for p in ph), 4),
                      "iters_ms": round(statistics.median(p[1] for p in ph), 4), "bitwise_same": same}), flush=True)
