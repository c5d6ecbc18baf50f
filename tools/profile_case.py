"""One warm solve of the C2 workload for ncu (`-k regex:solve_kernel`).
  python tools/profile_case.py [tau|fista|deblur]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fista"
op, basis, u0, meta = bench.make_inputs()
ctx = W.Context(0)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
if mode == "deblur":
    d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False), ctx)
    for _ in range(3):
        d.deblur(u0)
    print(d.last_stats())
else:
    x0 = W.analyze(u0, basis, ctx).values
    prob = W.DeblurProblem(W.SparseThetaOp(op, ctx), x0, w, 1e-4)
    cfg = dict(max_iters=100, tau=meta["tau"]) if mode == "fista" else dict(max_iters=0)
    for _ in range(3):
        r = W.fista(prob, P, W.SolverConfig(track_energy=False, **cfg), ctx)
    print(mode, r.wall_time_s * 1e3, "ms")
