"""Phase/barrier breakdown of the persistent solver from WBX_TRACE_FILE dumps.
  WBX_TRACE_FILE=/tmp/t.bin python tools/trace_phases.py run fista|tau ; python tools/trace_phases.py show /tmp/t.bin"""
import json
import os
import sys
from pathlib import Path

import numpy as np

if sys.argv[1] == "run":
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    from paper_1512_08401_b200 import waveblur as W
    op, basis, u0 = bench.make_inputs()
    meta = json.loads(bytes(np.load(bench.GOLDEN)["meta_json"]).decode())
    ctx = W.Context(0)
    P = W.spai(op, ctx)
    w = W.scale_weights(basis.layout)
    x0 = W.analyze(u0, basis, ctx).values
    prob = W.DeblurProblem(W.SparseThetaOp(op, ctx), x0, w, 1e-4)
    cfg = dict(max_iters=100, tau=meta["tau"]) if sys.argv[2] == "fista" else dict(max_iters=0)
    prec = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    for _ in range(3):
        r = W.fista(prob, P, W.SolverConfig(track_energy=False, precision=prec, **cfg), ctx)
    print("solve ms", r.wall_time_s * 1e3)
    sys.exit(0)

raw = np.fromfile(sys.argv[2], dtype=np.uint64)
G, cap = int(raw[0]), int(raw[1])
rec = 2 + cap * G * 2
last = raw[(len(raw) // rec - 1) * rec:][2:].reshape(cap, G, 2).astype(np.int64)
used = [i for i in range(cap) if last[i, :, 1].max() > 0]
arr = last[used]
t0 = arr[0, :, 0].min()
prev_release = None
phases, bars, skews = [], [], []
for i in range(len(used)):
    arrive, release = arr[i, :, 0], arr[i, :, 1]
    if prev_release is not None:
        phases.append((arrive.max() - prev_release.min()) / 1e3)
    bars.append((release.max() - arrive.max()) / 1e3)
    skews.append((arrive.max() - arrive.min()) / 1e3)
    prev_release = release
print(json.dumps({"grid": G, "barriers": len(used),
                  "phase_us(first..)": [round(x, 2) for x in phases[:8]],
                  "phase_us_median_even": round(float(np.median(phases[0::2])), 2) if phases else None,
                  "phase_us_median_odd": round(float(np.median(phases[1::2])), 2) if phases else None,
                  "barrier_us_median": round(float(np.median(bars)), 2),
                  "arrival_skew_us_median": round(float(np.median(skews)), 2)}))
if len(sys.argv) > 3 and sys.argv[3] == "blocks":
    # per-block work time of each phase (own arrival - own previous release), A = even, T = odd
    work = (arr[1:, :, 0] - arr[:-1, :, 1]) / 1e3
    out = {}
    for name, sl in (("A", work[0::2]), ("T", work[1::2])):
        m = sl.mean(axis=0)
        out[name] = {"p10": round(float(np.percentile(m, 10)), 2), "p50": round(float(np.median(m)), 2),
                     "p90": round(float(np.percentile(m, 90)), 2), "max": round(float(m.max()), 2),
                     "slowest": [int(b) for b in np.argsort(-m)[:12]],
                     "by_sm_pair": [round(float(x), 2) for x in m.reshape(-1, 2).mean(axis=1)[::16]]}
        # systematic vs random: the spread of the per-block MEAN work time vs the mean spread
        # within a phase (a block that is slow every phase can be rebalanced; noise cannot)
        out[name]["mean_spread_us"] = round(float(m.max() - m.min()), 2)
        out[name]["phase_spread_us_median"] = round(float(np.median(sl.max(axis=1) - sl.min(axis=1))), 2)
        out[name]["corr_first_second_half"] = round(float(np.corrcoef(sl[: len(sl) // 2].mean(0),
                                                                       sl[len(sl) // 2:].mean(0))[0, 1]), 3)
    print(json.dumps(out))
