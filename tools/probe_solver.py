"""Break the solve kernel's time into its phases (tau power iteration, FISTA loop,
init/decoupled) by running the public API with different configurations."""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

op, basis, u0, meta = bench.make_inputs()
ctx = W.Context(0)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
x0 = W.analyze(u0, basis, ctx).values
prob = W.DeblurProblem(W.SparseThetaOp(op, ctx), x0, w, 1e-4)
tau = meta["tau"]
out = {"blocks_per_sm_env": os.environ.get("WBX_SOLVER_BLOCKS_PER_SM")}
for name, cfg in [("init+decoupled (0 iters, tau given)", dict(max_iters=0, tau=tau)),
                  ("tau only (200 power iters)", dict(max_iters=0)),
                  ("fista 100 (tau given)", dict(max_iters=100, tau=tau)),
                  ("fista 100 + tau", dict(max_iters=100)),
                  ("fista 100 fp64 (tau given)", dict(max_iters=100, tau=tau, precision=64))]:
    ts = []
    for _ in range(4):
        r = W.fista(prob, P, W.SolverConfig(track_energy=False, **{"precision": 32, **cfg}), ctx)
        ts.append(r.wall_time_s * 1e3)
    out[name] = round(min(ts[1:]), 3)
print(json.dumps(out))
