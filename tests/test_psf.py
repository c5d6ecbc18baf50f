"""PSF generators, FFT convolution and degradation (operators.cpp:78-387)
against the reference's own outputs (tests/golden/psf_cases.npz, written by
oracle/make_psf_golden.py through the unmodified reference library).

* Analytic kernels (Gaussian, skewed Gaussian, Airy, defocus): host code in libwbx with the
  reference's expressions — bitwise, on CPU.
* Motion kernels (host curve + device FFT smoothing), convolve / apply_adjoint: bitwise
  against the oracle build (the device FFT restates its FFT arithmetic), GPU.
* add_noise / degrade: device Box-Muller with CUDA's log / cos (within 2 ulp of glibc): every
  pixel within 2 ulp of 1.0 of the reference, GPU."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_1512_08401_b200 import waveblur as W

G = np.load(Path(__file__).resolve().parent / "golden" / "psf_cases.npz")
INDEX = json.loads(bytes(G["index_json"]).decode())


def spec_of(s):
    kind, *v = s.split(":")
    if kind == "gaussian":
        return W.GaussianSpec(float(v[0]))
    if kind == "skewed":
        return W.SkewedGaussianSpec(float(v[0]))
    if kind == "motion":
        return W.MotionSpec(int(v[0]), float(v[1]), float(v[2]), int(v[3]))
    if kind == "airy":
        return W.AirySpec(float(v[0]))
    return W.DefocusSpec(float(v[0]))


ANALYTIC = [e for e in INDEX if not e["spec"].startswith("motion")]
MOTION = [e for e in INDEX if e["spec"].startswith("motion")]


@pytest.mark.parametrize("e", ANALYTIC, ids=[e["name"] for e in ANALYTIC])
def test_analytic_psf_bitwise(e):
    psf = W.generate_psf(spec_of(e["spec"]), e["dims"])
    assert W.psf_spec_string(psf.spec) == e["spec"]
    k = psf.kernel.ravel()
    if "sha256" in e:
        assert hashlib.sha256(k.tobytes()).hexdigest() == e["sha256"]
    else:
        assert np.array_equal(k, G["k_" + e["name"]])
    assert abs(k.sum() - 1.0) < 1e-12 and k.min() >= 0.0   # test_operators.cpp:46-60


def test_bad_psf_specs_rejected():  # test_operators.cpp:103-109
    with pytest.raises(W.BadSpec):
        W.generate_psf(W.GaussianSpec(-1.0), (32,))
    with pytest.raises(W.BadSpec):
        W.generate_psf(W.SkewedGaussianSpec(0.0), (32, 32))
    with pytest.raises(W.BadSpec):
        W.generate_psf(W.AirySpec(0.0), (32, 32))
    with pytest.raises(W.BadSpec):
        W.generate_psf(W.DefocusSpec(-2.0), (32, 32))
    with pytest.raises(W.ShapeMismatch):
        W.generate_psf(W.GaussianSpec(2.0), (48, 32))   # Image::require_dyadic


@pytest.mark.gpu
@pytest.mark.parametrize("e", MOTION, ids=[e["name"] for e in MOTION])
def test_motion_psf_bitwise(e):
    k = W.generate_psf(spec_of(e["spec"]), e["dims"]).kernel.ravel()
    assert np.array_equal(k, G["k_" + e["name"]])


@pytest.mark.gpu
def test_motion_psf_seed_determinism_and_errors():  # test_operators.cpp:92-101
    a = W.generate_psf(W.MotionSpec(5, 8.0, 1.0, 42), (64, 64)).kernel
    b = W.generate_psf(W.MotionSpec(5, 8.0, 1.0, 42), (64, 64)).kernel
    c = W.generate_psf(W.MotionSpec(5, 8.0, 1.0, 43), (64, 64)).kernel
    assert np.array_equal(a, b) and np.abs(a - c).max() > 0
    with pytest.raises(W.BadSpec):
        W.generate_psf(W.MotionSpec(1, 8.0, 1.0, 0), (32, 32))


@pytest.mark.gpu
def test_convolve_and_adjoint_bitwise():
    psf = W.generate_psf(W.MotionSpec(5, 8.0, 1.0, 42), (64, 64))
    u = G["scene64"].reshape(64, 64)
    assert np.array_equal(W.convolve(u, psf).ravel(), G["conv64"])
    assert np.array_equal(W.apply_adjoint_psf(u, psf).ravel(), G["adj64"])
    # adjointness <Hu, v> = <u, H*v> and constants preserved (test_operators.cpp:111-116)
    v = np.random.default_rng(3).standard_normal((64, 64))
    lhs = np.vdot(W.convolve(u, psf), v)
    rhs = np.vdot(u, W.apply_adjoint_psf(v, psf))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    c = W.convolve(np.full((64, 64), 0.37), psf)
    assert np.allclose(c, 0.37, rtol=1e-12, atol=0)


@pytest.mark.gpu
def test_degrade_and_noise_vs_reference():
    psf = W.generate_psf(W.MotionSpec(5, 8.0, 1.0, 42), (64, 64))
    u = G["scene64"].reshape(64, 64)
    ulp2 = 2 * np.spacing(1.0)
    n = W.add_noise(u, 1e-2, 11).ravel()
    assert np.abs(n - G["noise64"]).max() <= ulp2 and np.mean(n == G["noise64"]) > 0.95
    d = W.degrade(u, W.DegradationModel(psf, 1e-2, 11)).ravel()
    assert np.abs(d - G["degrade64"]).max() <= ulp2 and np.mean(d == G["degrade64"]) > 0.95
    assert np.array_equal(W.add_noise(u, 0.0, 11), u)
    with pytest.raises(W.BadSpec):
        W.add_noise(u, -1.0, 1)
