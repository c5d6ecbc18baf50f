"""Which engine the C3 (1024^2 spatially varying) operator gets, and why (WBX_VERBOSE=1)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
lad = W.SigmaLadder.from_npz(np.load(ROOT / "tests" / "golden" / "c3_ladder_1024.npz"))
op = W.theta_varying(lad, 2.5, 7.5)
ctx = W.Context(0)
basis = W.make_basis(W.FilterFamily.Daubechies, 4, (1024, 1024), 4)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False), ctx)
print(d.kernels(), op.nnz(), op.info(ctx).nonempty_rows, op.info(ctx).nonempty_cols)
import json  # noqa: E402
for _ in range(3):
    u, rep = d.deblur(np.zeros(op.n) + 0.5, clamp=True)
print(json.dumps({"tau_ms": d.phase_ms()[0], "iters_ms": d.phase_ms()[1], "tau_stats": d.tau_stats()}))
