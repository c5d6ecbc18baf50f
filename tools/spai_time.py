"""Time SPAI (Gram diagonals on the device) at the C2 operator."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1512_08401_b200 import waveblur as W  # noqa: E402

op, basis, u0 = bench.make_inputs()
ctx = W.Context(0)
op.device(ctx)
for _ in range(3):
    t0 = time.perf_counter()
    P = W.spai(op, ctx)
    t1 = time.perf_counter()
print("spai ms (incl. CSC build + uploads)", round((t1 - t0) * 1e3, 1))
