"""B200-native hot path of waveblur (Escande & Weiss, arXiv:1512.08401).

`waveblur` mirrors the reference's C++ API (analyze/synthesize, spmv/spmv_t, the
weighted soft-threshold prox, estimate_step, ista/fista) over the C ABI of libwbx.so
(include/wbx.h): hand-written sm_100a kernels, no CPU fallback.
"""
from . import waveblur  # noqa: F401  (loads libwbx.so; raises if it is missing)

__all__ = ["waveblur"]
