import ctypes as C, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["WBX_DEBUG_MODE"] = "2"
import bench
from paper_1512_08401_b200 import waveblur as W
from paper_1512_08401_b200 import _native as N
N.lib.wbx_diag_slice_profile.argtypes = [C.POINTER(C.c_double)]
op, basis, u0, meta = bench.make_inputs()
ctx = W.Context(0)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
x0 = W.analyze(u0, basis, ctx).values
prob = W.DeblurProblem(W.SparseThetaOp(op, ctx), x0, w, 1e-4)
out = (C.c_double * 6)()
for name, cfg in [("fista", dict(max_iters=100, tau=meta["tau"])), ("tau", dict(max_iters=0))]:
    W.fista(prob, P, W.SolverConfig(track_energy=False, **cfg), ctx)
    N.lib.wbx_diag_slice_profile(out)
    r = W.fista(prob, P, W.SolverConfig(track_energy=False, **cfg), ctx)
    N.lib.wbx_diag_slice_profile(out)
    print(name, "ms", round(r.wall_time_s * 1e3, 3), "cycles/slice: tma_wait %.0f gather+fma %.0f combine %.0f issue %.0f post %.0f slices %.0f" % tuple(out))
