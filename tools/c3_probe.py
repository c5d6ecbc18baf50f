import sys, numpy as np
sys.path.insert(0,'/root/repo')
from pathlib import Path
from paper_1512_08401_b200 import waveblur as W
import bench
lad = W.SigmaLadder.from_npz(np.load(Path('/root/repo/tests/golden/c3_ladder_1024.npz')))
opv = W.theta_varying(lad, 2.5, 7.5)
op, basis, u0, meta = bench.make_inputs()
ctx=W.Context(0)
P=W.spai(opv, ctx); w=W.scale_weights(basis.layout)
d=W.Deblurrer(opv, basis, P, w, 1e-4, W.SolverConfig(max_iters=100, track_energy=False), ctx)
for _ in range(3): d.deblur(u0)
print(d.phase_ms(), d.tau_stats())
