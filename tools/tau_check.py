"""tau on the fp32 hot path (Lanczos by default, WBX_TAU=power for the literal power
iteration) against the reference's tau on the golden operators: value, the reference's
iteration count, device time of the estimate."""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import importlib.util  # noqa: E402
_spec = importlib.util.spec_from_file_location("wbx_conftest", Path(__file__).resolve().parents[1] / "tests" / "conftest.py")
_conf = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_conf)
Golden = _conf.Golden
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

out = {"WBX_TAU": os.environ.get("WBX_TAU", "lanczos")}
for name in ["c1_db4_256", "c1_sym6_256", "s64_sym6_spai", "s128_1d_sym6", "s32_sym4_naive", "c2_db4_1024"]:
    g = Golden(name)
    op = g.operator()
    b = W.make_basis(W.FilterFamily(g.family), g.meta["order"], g.dims, g.meta["J"])
    x0 = np.zeros(op.n)
    kind = g.meta["precond"]
    if kind == "spai":
        P = W.spai(op)
    elif kind == "jacobi":
        gd = W.gram_diagonals(op)
        P = W.jacobi(op, max(1e-3 * gd.diagM.max(), 1e-300))
    else:
        P = W.identity_precond(op.n)
    prob = W.DeblurProblem(W.SparseThetaOp(op), x0, g.weights(), g.meta["lambda"])
    ts = []
    for _ in range(4):
        r = W.fista(prob, P, W.SolverConfig(max_iters=0, precision=32, track_energy=False))
        ts.append(r.wall_time_s * 1e3)
    out[name] = {"tau_rel_err": abs(r.tau - g.meta["tau"]) / g.meta["tau"], "iters": r.tau_iters,
                 "ref_iters": g.meta.get("tau_iters"), "ms": round(min(ts[1:]), 3)}
print(json.dumps(out, indent=1))
