"""Wall time of the drop-in fista() (wbx_pgd) at C2: setup vs solve (tracked / untracked, K = 0 / 100)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

op, basis, u0 = bench.make_inputs()
ctx = W.Context(0)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
x0 = W.analyze(u0, basis, ctx).values
prob = W.DeblurProblem(W.SparseThetaOp(op, ctx), x0, w, 1e-4)
out = {}
for name, cfg in [("untracked_k0", W.SolverConfig(max_iters=0, track_energy=False)),
                  ("untracked_k100", W.SolverConfig(max_iters=100, track_energy=False)),
                  ("tracked_k0", W.SolverConfig(max_iters=0, track_energy=True)),
                  ("tracked_k100", W.SolverConfig(max_iters=100, track_energy=True))]:
    W.fista(prob, P, cfg, ctx)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        W.fista(prob, P, cfg, ctx)
        ts.append(1e3 * (time.perf_counter() - t0))
    out[name] = round(float(np.median(ts)), 3)
print(json.dumps(out))
