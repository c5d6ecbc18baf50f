"""A small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): the C1
golden deblur on the window engine (fp32, tracked and untracked), the fp64 stream engine,
the standalone SpMV kernels, the sharded engine at world 2 and the PSF / FFT path, at sizes
that finish under the sanitizer in minutes.
  compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

z = np.load(ROOT / "tests" / "golden" / "s64_sym6_spai.npz")
meta = json.loads(bytes(z["meta_json"]).decode())
gl = W.GeneratorList(tuple(meta["dims"]), meta["J"], W.FilterFamily.Symmlet, 6, z["gen_block"].astype(np.uint32),
                     z["gen_index"].astype(np.uint32), z["gen_count"].astype(np.uint64), z["gen_value"])
op = W.theta_from_generators(gl)
basis = W.make_basis(W.FilterFamily.Symmlet, 6, tuple(meta["dims"]), meta["J"])
ctx = W.Context(0)
P = W.spai(op, ctx)
w = W.scale_weights(basis.layout)
u0 = z["u0"].reshape(meta["dims"])
iters = 20
for cfg in (W.SolverConfig(max_iters=iters, track_energy=False),
            W.SolverConfig(max_iters=iters, track_energy=True, track_support=True),
            W.SolverConfig(max_iters=iters, track_energy=False, precision=64)):
    d = W.Deblurrer(op, basis, P, w, 1e-4, cfg, ctx)
    u, rep = d.deblur(u0, clamp=True)
    print(d.kernels(), rep.iters_used, float(np.abs(u).sum()))
x = np.random.default_rng(0).standard_normal(op.n)
print(float(np.abs(W.spmv(op, x, ctx)).sum()), float(np.abs(W.spmv_t(op, x, ctx)).sum()))
psf = W.generate_psf(W.MotionSpec(5, 8.0, 1.0, 3), tuple(meta["dims"]), ctx)
print(float(W.degrade(u0, W.DegradationModel(psf, 1e-2, 1), ctx).sum()))
import torch  # noqa: E402
from paper_1512_08401_b200.sharded import ShardedDeblurrer  # noqa: E402
sh = ShardedDeblurrer(ctx, op, basis, P, w, 1e-4, iters, 2, [0, 1], tau=rep.tau)
dev = torch.device("cuda", 0)
ud = torch.from_numpy(u0.ravel().copy()).to(dev)
out = torch.empty_like(ud)
sh.deblur_dev(ud.data_ptr(), out.data_ptr())
ctx.synchronize()
print("sharded", float(out.abs().sum()))
print("SANITIZE_CASE_OK")
