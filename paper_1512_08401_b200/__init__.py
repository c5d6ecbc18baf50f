"""B200-native hot path of waveblur (Escande & Weiss, arXiv:1512.08401).

`waveblur` mirrors the reference's C++ API (analyze/synthesize, spmv/spmv_t, the
weighted soft-threshold prox, estimate_step, ista/fista) over the C ABI of libwbx.so
(include/wbx.h): hand-written sm_100a kernels, no CPU fallback. Importing `waveblur`
(or `_native`) loads libwbx.so and raises if it is missing; the package itself loads
nothing, so host-only helpers (`synthetic`) import without the native library.
"""
import importlib

__all__ = ["waveblur"]


def __getattr__(name):
    if name in ("waveblur", "sharded", "synthetic", "sharding", "_native"):
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
