"""Synthetic inputs of the reference's shapes (host-side, numpy; not on the hot path).

Mirrors the reference's fixture generators so bench inputs have the reference's
statistics: `synthetic_scene` (image.cpp:185-221), the Gaussian PSF
(operators.cpp:98-117, wrapped coordinates, unit mass), circular convolution
(operators.cpp:70-77; numpy FFT instead of FFTW) and `add_noise` (operators.cpp:344-356,
counter-based splitmix64 + per-index Box-Muller). The reference's own degrade() output
for the 256^2 fixture is committed under tests/golden and checked against this module.
"""
from __future__ import annotations

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def rng_at(seed: int, i: np.ndarray) -> np.ndarray:
    """CounterRng::at (rng.hpp:17-22), vectorised (uint64 wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + _GOLD * (i.astype(np.uint64) + np.uint64(1))
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _u01(v: np.ndarray) -> np.ndarray:
    return ((v >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53


def synthetic_scene(dims) -> np.ndarray:
    dims = tuple(int(d) for d in dims)
    if len(dims) == 1:
        n = dims[0]
        t = np.arange(n) / n
        v = 0.35 + 0.25 * np.sin(2.0 * np.pi * 3.0 * t)
        v = np.where((t > 0.2) & (t < 0.3), v + 0.4, v)
        v = np.where((t > 0.55) & (t < 0.57), 1.0, v)
        v = v + 0.15 * np.exp(-(((t - 0.8) / 0.03) ** 2))
        return np.clip(v, 0.0, 1.0)
    h, w = dims
    y = (np.arange(h) / h)[:, None]
    x = (np.arange(w) / w)[None, :]
    v = 0.25 + 0.2 * np.sin(2.0 * np.pi * 2.0 * x) * np.cos(2.0 * np.pi * 1.5 * y)
    d1 = np.hypot(x - 0.3, y - 0.35)
    v = np.where(d1 < 0.16, v + 0.45 * (1.0 - d1 / 0.16), v)
    v = np.where(np.hypot(x - 0.72, y - 0.65) < 0.1, v + 0.5, v)
    k = (x * 24.0).astype(np.int64)
    v = np.where((y > 0.82) & (y < 0.92) & (k % 2 == 0), v + 0.4, v)
    v = np.where((np.abs((x - y) * w) < 1.5) & (x > 0.05) & (x < 0.5), 0.95, v)
    return np.clip(v, 0.0, 1.0)


def gaussian_psf(dims, sigma: float) -> np.ndarray:
    dims = tuple(int(d) for d in dims)
    if sigma < 1.0:
        k = np.zeros(dims)
        k.flat[0] = 1.0
        return k
    coords = [np.where(np.arange(n) < n // 2, np.arange(n), np.arange(n) - n).astype(np.float64)
              for n in dims]
    if len(dims) == 1:
        k = np.exp(-coords[0] ** 2 / (2.0 * sigma * sigma))
    else:
        t1, t2 = np.meshgrid(coords[0], coords[1], indexing="ij")
        k = np.exp(-(t1 * t1 + t2 * t2) / (2.0 * sigma * sigma))
    return k / k.sum()


def convolve(u: np.ndarray, kernel: np.ndarray) -> np.ndarray:
    return np.real(np.fft.ifftn(np.fft.fftn(u) * np.fft.fftn(kernel)))


def add_noise(u: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    if sigma == 0.0:
        return u.copy()
    i = np.arange(u.size, dtype=np.uint64)
    u1 = _u01(rng_at(seed, 2 * i))
    u2 = _u01(rng_at(seed, 2 * i + np.uint64(1)))
    b = sigma * np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return u + b.reshape(u.shape)


def degrade(dims, sigma: float = 5.0, noise: float = 5e-3, seed: int = 2024):
    """observed = add_noise(convolve(scene, gaussian(sigma)), noise, seed); returns (clean, observed)."""
    clean = synthetic_scene(dims)
    obs = add_noise(convolve(clean, gaussian_psf(dims, sigma)), noise, seed)
    return clean, obs


def psnr(u: np.ndarray, v: np.ndarray) -> float:
    mse = float(np.mean((u - v) ** 2))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(1.0 / mse)
