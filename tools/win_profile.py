"""Cycle accounting of the window engine (needs the diagnostics build):
  make -C paper_1512_08401_b200 prof && WBX_LIB=paper_1512_08401_b200/lib/libwbx_prof.so python tools/win_profile.py
Per warp and phase of each side (A = Theta rows, T = Theta^T rows), in SM cycles: window
fill, slice loop, grid barrier (incl. waiting for the slowest CTA)."""
import ctypes as C
import json

import numpy as np
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1512_08401_b200 import _native  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

lib = _native.lib
lib.wbx_diag_slice_profile.argtypes = [C.POINTER(C.c_double)]
op, basis, u0 = bench.make_inputs()
meta = json.loads(bytes(np.load(bench.GOLDEN)["meta_json"]).decode())
ctx = W.Context(0)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
x0 = W.analyze(u0, basis, ctx).values
prob = W.DeblurProblem(W.SparseThetaOp(op, ctx), x0, w, 1e-4)
buf = (C.c_double * 8)()
res = {}
for name, cfg, phases in [("fista", dict(max_iters=100, tau=meta["tau"]), 200), ("tau", dict(max_iters=0), None)]:
    W.fista(prob, P, W.SolverConfig(track_energy=False, precision=32, **cfg), ctx)
    lib.wbx_diag_slice_profile(buf)  # reset
    r = W.fista(prob, P, W.SolverConfig(track_energy=False, precision=32, **cfg), ctx)
    lib.wbx_diag_slice_profile(buf)
    h = list(buf)
    # phases of each side (the Lanczos tau takes fewer product pairs than the reference's
    # iteration count: pass them as argv[1], WBX_VERBOSE=1 prints them)
    nph = phases // 2 if phases else (int(sys.argv[1]) if len(sys.argv) > 1 else r.tau_iters)
    warps = 296 * 8
    per = warps * nph
    res[name] = {"ms": round(r.wall_time_s * 1e3, 3), "phases": nph,
                 "A": {"fill": round(h[0] / per), "loop": round(h[1] / per),
                       "barrier": round(h[2] / per)},
                 "T": {"fill": round(h[3] / per), "loop": round(h[4] / per),
                       "barrier": round(h[5] / per)}}
print(json.dumps(res))
