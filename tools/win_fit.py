"""Fit the window engine's balance cost model to measured per-CTA phase times (C2).

For each round: build the operator's window layout under the current model, trace one FISTA
solve (WBX_TRACE_FILE: per-CTA arrival stamps per barrier), take each CTA's mean phase-A and
phase-T work time, and its layout features (wbx_diag_win_features); fit per side by
non-negative least squares
    t_cta = k0 + a*sum(1/m) + b*sum(nq/m) + c*sum((q-1)/m) + d*nnz + e*rows
i.e. cost(row) = (a + b nq + c (q-1))/m + d len + e (winlayout.cu balance()), refit on the data
of every round so far, and report the untraced deblur time of each model.
  python tools/win_fit.py [rounds]"""
import ctypes as C
import json
import os
import statistics
import sys
import tempfile
from pathlib import Path

import numpy as np
from scipy.optimize import nnls

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1512_08401_b200 import _native as N  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
z = np.load(bench.GOLDEN)
meta = json.loads(bytes(z["meta_json"]).decode())
_, basis, u0 = bench.make_inputs()
ctx = W.Context(0)
dev = torch.device("cuda", 0)
stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
with torch.cuda.stream(stream):
    u = torch.from_numpy(u0.ravel().copy()).to(dev)
    out = torch.empty_like(u)
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)


def fresh_op():
    gl = W.GeneratorList(bench.DIMS, 4, W.FilterFamily.Daubechies, 4, z["gen_block"].astype(np.uint32),
                         z["gen_index"].astype(np.uint32), z["gen_count"].astype(np.uint64), z["gen_value"])
    return W.theta_from_generators(gl)


def per_block(path):
    raw = np.fromfile(path, dtype=np.uint64)
    G, cap = int(raw[0]), int(raw[1])
    rec = 2 + cap * G * 2
    last = raw[(len(raw) // rec - 1) * rec:][2:].reshape(cap, G, 2).astype(np.int64)
    used = [i for i in range(cap) if last[i, :, 1].max() > 0]
    arr = last[used]
    work = (arr[1:, :, 0] - arr[:-1, :, 1]) / 1e3
    return work[0::2].mean(axis=0), work[1::2].mean(axis=0)  # A, T


def measure(model):
    for side in "AT":
        if model[side] is None:
            os.environ.pop(f"WBX_WIN_MODEL_{side}", None)
        else:
            os.environ[f"WBX_WIN_MODEL_{side}"] = ",".join(f"{v:.6g}" for v in model[side])
    op = fresh_op()
    P = W.spai(op, ctx)
    w = W.scale_weights(basis.layout)
    with tempfile.TemporaryDirectory() as td:
        os.environ["WBX_TRACE_FILE"] = str(Path(td) / "t.bin")
        d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False, tau=meta["tau"]),
                        ctx)
        for _ in range(2):
            d.deblur(u0)
        tA, tT = per_block(os.environ["WBX_TRACE_FILE"])
        del os.environ["WBX_TRACE_FILE"]
    feats = []
    for side in (0, 1):
        G = C.c_int()
        buf = np.zeros(2048 * 6)
        W._check(N.lib.wbx_diag_win_features(d.handle, side, W._dptr(buf), C.byref(G)))
        feats.append(buf[: G.value * 6].reshape(G.value, 6))
    del d
    # untraced timing of the full deblur (graphs on)
    d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False), ctx)
    for _ in range(3):
        d.deblur_dev(u.data_ptr(), out.data_ptr())
    ms = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.zero_()
            a.record(stream)
        d.deblur_dev(u.data_ptr(), out.data_ptr())
        with torch.cuda.stream(stream):
            b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    ph = d.phase_ms()
    return tA, tT, feats, statistics.median(ms), ph


def design(F):  # columns: 1, sum 1/m, sum nq/m, sum (q-1)/m, nnz, rows
    return np.column_stack([np.ones(len(F)), F[:, 1], F[:, 2], F[:, 3], F[:, 4], F[:, 0]])


data = {"A": [], "T": []}
model = {"A": None, "T": None}
for r in range(rounds + 1):
    tA, tT, feats, ms, ph = measure(model)
    print(json.dumps({"round": r, "model": {k: (None if v is None else [round(x, 5) for x in v]) for k, v in model.items()},
                      "deblur_ms": round(ms, 4), "tau_ms": round(ph[0], 4), "iters_ms": round(ph[1], 4),
                      "A_spread_us": round(float(tA.max() - tA.min()), 3), "A_max_us": round(float(tA.max()), 3),
                      "T_spread_us": round(float(tT.max() - tT.min()), 3), "T_max_us": round(float(tT.max()), 3)}),
          flush=True)
    data["A"].append((feats[0], tA))
    data["T"].append((feats[1], tT))
    for side in "AT":
        X = np.vstack([design(F) for F, _ in data[side]])
        y = np.concatenate([t for _, t in data[side]])
        coef, _ = nnls(X, y)
        model[side] = list(coef[1:])  # the constant k0 does not move the partition
        resid = y - X @ coef
        print(json.dumps({"side": side, "k0": round(float(coef[0]), 4), "coef": [round(float(c), 6) for c in coef[1:]],
                          "rms_us": round(float(np.sqrt(np.mean(resid ** 2))), 4)}), flush=True)
