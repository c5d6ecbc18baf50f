"""Cycle accounting of the stencil engine's FISTA kernel (needs the diagnostics build):
  make -C paper_1512_08401_b200 prof && WBX_STENCIL=1 WBX_LIB=paper_1512_08401_b200/lib/libwbx_prof.so python tools/st_profile.py
Per warp and phase (A = Theta, T = Theta^T), in SM cycles: window fill (issue to mbarrier),
warp entries (taps), part sums + epilogue, grid barrier (incl. waiting for the slowest CTA)."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

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
cfg = W.SolverConfig(track_energy=False, precision=32, max_iters=100, tau=meta["tau"])
W.fista(prob, P, cfg, ctx)
lib.wbx_diag_slice_profile(buf)  # reset
r = W.fista(prob, P, cfg, ctx)
lib.wbx_diag_slice_profile(buf)
h = list(buf)
per = 296 * 8 * 100
names = ["fill", "taps", "epilogue", "barrier"]
print(json.dumps({"ms": round(r.wall_time_s * 1e3, 3),
                  "A": {n: round(h[i] / per) for i, n in enumerate(names)},
                  "T": {n: round(h[4 + i] / per) for i, n in enumerate(names)}}))
