"""Lanczos step-estimate sweep at C2: first check m, agreement tolerance -> tau, its deviation
from the reference's tau (golden), the reference iteration count, Lanczos steps, device ms.
  python tools/lz_sweep.py"""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

op, basis, u0 = bench.make_inputs()
meta = json.loads(bytes(np.load(bench.GOLDEN)["meta_json"]).decode())
ctx = W.Context(0)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
CASES = [(60, 4, 4, "1e-12"), (52, 4, 4, "1e-9"), (48, 4, 4, "1e-8"), (44, 4, 4, "1e-8"), (40, 4, 4, "1e-8"),
         (48, 4, 4, "1e-9"), (44, 4, 4, "1e-9"), (40, 4, 4, "1e-9"), (36, 4, 4, "1e-9"), (40, 4, 4, "1e-10"),
         (48, 4, 4, "1e-10"), (56, 4, 4, "1e-12"), (32, 4, 4, "1e-8")]
for first, every, gap, tol in CASES:
    os.environ.update(WBX_LZ_FIRST=str(first), WBX_LZ_EVERY=str(every), WBX_LZ_GAP=str(gap), WBX_LZ_TOL=tol)
    d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False), ctx)
    ts = []
    for _ in range(5):
        _, rep = d.deblur(u0, clamp=True)
        ts.append(d.phase_ms()[0])
    tau, iters, steps = d.tau_stats()
    print(json.dumps({"first": first, "tol": tol, "tau": tau, "rel_dev": abs(tau - meta["tau"]) / meta["tau"],
                      "ref_iters": iters, "steps": steps, "tau_ms": round(float(np.median(ts)), 4)}), flush=True)
