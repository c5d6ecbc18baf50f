"""Warm runs of the C2 workload for ncu (`-k regex:...`): the deblur unit (the bench step:
tau + FISTA + DWT/IDWT) and the tracked fista() of the drop-in binding.
  python tools/profile_case.py [deblur|tracked|both|c5]   (c5: one batch of 8 images)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "both"
op, basis, u0 = bench.make_inputs()
ctx = W.Context(0)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
if mode in ("deblur", "both"):
    d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False), ctx)
    for _ in range(2):
        d.deblur(u0)
    print("deblur", d.last_stats())
if mode == "c5":
    import numpy as np
    from paper_1512_08401_b200 import synthetic as S
    imgs = np.stack([S.degrade(bench.DIMS, 5.0, 5e-3, s)[1] for s in range(8)])
    d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False), ctx, batch=8)
    for _ in range(2):
        d.deblur(imgs)
    print("c5", d.kernels(), d.last_stats())
if mode in ("tracked", "both"):
    x0 = W.analyze(u0, basis, ctx).values
    prob = W.DeblurProblem(W.SparseThetaOp(op, ctx), x0, w, 1e-4)
    for _ in range(2):
        r = W.fista(prob, P, W.SolverConfig(max_iters=100, track_energy=True), ctx)
    print("tracked", r.wall_time_s * 1e3, "ms")
