"""C5 timing probe: 64 images of the C2 operator in batches of 8 (inputs resident, one L2 flush),
with the engine the solver picks (WBX_CIRC_SLOTS / WBX_ENGINE change it). Prints images/s."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

op, basis, u0 = bench.make_inputs()
ctx = W.Context(0)
dev = torch.device("cuda:0")
stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
r = bench.run_c5(W, torch, ctx, stream, dev, op, basis, P, w, flush, 0, 1)
d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False), ctx, batch=8)
r["kernels"] = d.kernels()
print(json.dumps(r))
