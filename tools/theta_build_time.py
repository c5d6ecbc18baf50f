"""Time the device Theta_K construction (build_theta_conv + weighted top-K) at C2 and 4096^2."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

ctx = W.Context(0)
for side in (1024, 4096):
    dims = (side, side)
    basis = W.make_basis(W.FilterFamily.Daubechies, 4, dims, 4)
    psf = W.gaussian_psf_kernel(dims, 5.0)
    w = W.dyadic_band_weights(basis.layout)
    K = 3 * side * side
    for _ in range(2):
        t0 = time.perf_counter()
        gl = W.theta_conv_topk(basis, psf, K, w, ctx)
        t1 = time.perf_counter()
    t2 = time.perf_counter()
    op = W.theta_from_generators(gl)
    t3 = time.perf_counter()
    print(f"{side}^2: theta_conv_topk {1e3 * (t1 - t0):.1f} ms ({gl.blocks.size} groups), "
          f"CSR expand {1e3 * (t3 - t2):.1f} ms, nnz {op.nnz()}")
