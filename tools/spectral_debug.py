"""Spectral FISTA vs the window engine on a small operator: x after K iterations (debug aid)."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1512_08401_b200 import synthetic as S  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

dims, fam, order, J, sigma, kf = (64, 64), W.FilterFamily.Haar, 1, 1, 3.0, 4
if len(sys.argv) > 1:
    dims = (int(sys.argv[1]),) * 2
    J = int(sys.argv[2])
basis = W.make_basis(fam, order, dims, J)
n = basis.layout.total()
psf = W.gaussian_psf_kernel(dims, sigma)
op = W.theta_from_generators(W.theta_conv_topk(basis, psf, kf * n, W.dyadic_band_weights(basis.layout)))
P = W.spai(op)
clean = S.synthetic_scene(dims)
u0 = S.add_noise(W.synthesize(W.spmv(op, W.analyze(clean, basis).values), basis), 5e-3, 9)
w = W.scale_weights(basis.layout)
x0 = W.analyze(u0, basis).values
prob = W.DeblurProblem(W.SparseThetaOp(op), x0, w, 1e-4)
colnz = np.zeros(n, bool)
colnz[op.col_indices] = True
for K in (0, 1, 2, 5):
    os.environ.pop("WBX_ENGINE", None)
    a = W.fista(prob, P, W.SolverConfig(max_iters=K, precision=32, track_energy=False))
    os.environ["WBX_ENGINE"] = "window"
    b = W.fista(prob, P, W.SolverConfig(max_iters=K, precision=32, track_energy=False))
    d = np.abs(a.x_final - b.x_final)
    print(K, "tau", a.tau, b.tau, "C max diff", d[colnz].max(), "dec max diff", d[~colnz].max(),
          "|x| C", np.abs(b.x_final[colnz]).max(), "nC", colnz.sum())
