"""Lanczos tau (fp32 hot path, default) vs the literal fp32 power iteration (WBX_TAU=power) and
the fp64 reference-mode estimate on random sparse operators: reference iteration count and tau.
  python tools/tau_stress.py [count]"""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1512_08401_b200 import waveblur as W  # noqa: E402


def random_op(rng, n, per_row):
    rows = []
    for r in range(n):
        k = rng.integers(0, per_row + 1)
        cols = np.sort(rng.choice(n, size=k, replace=False)) if k else np.zeros(0, np.int64)
        rows.append(cols)
    ro = np.zeros(n + 1, np.uint64)
    ro[1:] = np.cumsum([len(c) for c in rows])
    ci = np.concatenate(rows).astype(np.uint32) if ro[-1] else np.zeros(0, np.uint32)
    vals = rng.standard_normal(int(ro[-1])) * rng.uniform(0.1, 2.0)
    return W.SparseOperator(n, ro, ci, vals)


count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(1234)
res = []
for t in range(count):
    n = int(rng.choice([64, 256, 1024, 4096]))
    op = random_op(rng, n, int(rng.integers(1, 12)))
    p = rng.uniform(0.2, 3.0, n)
    P = W.DiagonalPreconditioner(p, W.PrecondKind.Spai)
    prob = W.DeblurProblem(W.SparseThetaOp(op), np.zeros(n), np.ones(n), 1e-4)
    cfg = W.SolverConfig(max_iters=0, precision=32, track_energy=False)
    os.environ.pop("WBX_TAU", None)
    lz = W.fista(prob, P, cfg)
    os.environ["WBX_TAU"] = "power"
    pw = W.fista(prob, P, cfg)
    os.environ.pop("WBX_TAU", None)
    t64, it64 = W.estimate_step(W.SparseThetaOp(op), P, cfg.step_safety, return_iters=True)
    res.append({"n": n, "nnz": int(op.nnz()), "iters_lz": lz.tau_iters, "iters_pw": pw.tau_iters, "iters_64": it64,
                "rel_lz": abs(lz.tau - t64) / t64, "rel_pw": abs(pw.tau - t64) / t64})
bad = [r for r in res if r["iters_lz"] != r["iters_64"] or r["rel_lz"] > 1e-6]
print(json.dumps({"cases": len(res), "mismatch_lz": len(bad),
                  "mismatch_pw": sum(r["iters_pw"] != r["iters_64"] or r["rel_pw"] > 1e-6 for r in res),
                  "max_rel_lz": max(r["rel_lz"] for r in res), "max_rel_pw": max(r["rel_pw"] for r in res),
                  "bad": bad[:10]}, indent=1))
