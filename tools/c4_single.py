"""C4 operator (4096^2 varying) through the single-GPU Deblurrer (no sharding): which engine
runs and how fast, vs the row-sharded path at world 1."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1512_08401_b200 import synthetic as S  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dims = (size, size)
ROOT = Path(__file__).resolve().parents[1]
t0 = time.perf_counter()
lad = W.SigmaLadder.from_npz(np.load(ROOT / "tests" / "golden" / "c3_ladder_1024.npz"))
if size != 1024:
    lad = W.SigmaLadder(lad.sigmas, [W.rescale_generators(g, dims) for g in lad.levels])
op = W.theta_varying(lad, 2.5, 7.5)
ctx = W.Context(0)
basis = W.make_basis(W.FilterFamily.Daubechies, 4, dims, 4)
clean = S.synthetic_scene(dims)
u0 = S.add_noise(W.synthesize(W.spmv(op, W.analyze(clean, basis, ctx).values, ctx), basis, ctx), 5e-3, 2024)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
t1 = time.perf_counter()
d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False), ctx)
t2 = time.perf_counter()
dev = torch.device("cuda", 0)
u = torch.from_numpy(u0.ravel().copy()).to(dev)
out = torch.empty_like(u)
for _ in range(2):
    d.deblur_dev(u.data_ptr(), out.data_ptr(), clamp=True)
ctx.synchronize()
ts = []
for _ in range(3):
    a = time.perf_counter()
    d.deblur_dev(u.data_ptr(), out.data_ptr(), clamp=True)
    ctx.synchronize()
    ts.append(1e3 * (time.perf_counter() - a))
print({"size": size, "setup_s": round(t1 - t0, 1), "solver_create_s": round(t2 - t1, 1), "ms": round(min(ts), 2),
       "phase_ms": d.phase_ms() if hasattr(d, "phase_ms") else None, "nnz": op.nnz()})
