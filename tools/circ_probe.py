"""Step-estimate time at C2 (1024^2 stationary): block-Fourier (default) vs Lanczos
(WBX_TAU=lanczos). Prints tau, its iteration count and the device ms of the estimate."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

z = np.load(ROOT / "tests" / "golden" / "c2_db4_1024.npz")
gl = W.GeneratorList((1024, 1024), 4, W.FilterFamily.Daubechies, 4, z["gen_block"].astype(np.uint32),
                     z["gen_index"].astype(np.uint32), z["gen_count"].astype(np.uint64), z["gen_value"])
op = W.theta_from_generators(gl)
ctx = W.Context(0)
basis = W.make_basis(W.FilterFamily.Daubechies, 4, (1024, 1024), 4)
P = W.spai(op, ctx)
d = W.Deblurrer(op, basis, P, W.scale_weights(basis.layout), 1e-4,
                W.SolverConfig(max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 0, track_energy=False), ctx)
ts = []
for _ in range(8):
    u, rep = d.deblur(np.zeros(op.n) + 0.5, clamp=True)
    ts.append(d.phase_ms())
print(json.dumps({"kernels": d.kernels(), "tau": rep.tau, "tau_iters": rep.tau_iters, "tau_iters_ms": ts}))
