"""The reference's own doctest suites (proj/tests/test_{wavelet,operators,theta,precond,solver}.cpp),
unmodified, with the reference's hot path routed to libwbx.so by the maintainer binding of
INTEGRATION.md §2 (integration/wbx_backend.cpp; `make -C oracle wbx-tests` links it ahead of
the reference objects, whose routed definitions are renamed to *_host). Every analyze /
synthesize / spmv / spmv_t / approx_gradient / energy / prox / estimate_step / ista / fista /
gram_diagonals / jacobi / spai call of those suites on a SparseThetaOp or ExactThetaOp, and every
generate_psf / convolve / apply_adjoint / add_noise / degrade call, runs through libwbx (the B200),
in the fp64 mode, at the suites' native tolerances (bitwise where they compare bitwise).

The binaries are built in the build container (they compile the reference's test sources
from /root/reference) and travel prebuilt under oracle/_ref/."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"
SUITES = ["wavelet", "operators", "theta", "precond", "solver"]

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_through_libwbx(suite):
    exe = REF / f"wbx_test_{suite}"
    if not exe.exists():
        pytest.skip(f"{exe.name} not built (make -C oracle wbx-tests needs /root/reference)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900, cwd=REF)
    out = r.stdout + r.stderr
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out)
    assert m, out[-2000:]
    assert int(m.group(3)) == 0 and r.returncode == 0, out[-4000:]
    assert int(m.group(1)) == int(m.group(2)) > 0


@pytest.mark.parametrize("precision", ["64", "32"])
def test_reference_acceptance_through_libwbx(precision):
    """acceptance.cpp criteria 1-8 with the hot path on the B200. Criterion 9
    compares CSV output of the reference CLI across thread counts; the CLI needs CLI11 and
    nlohmann/json, which are not in this image, so it cannot run here (nor upstream of it)."""
    exe = REF / "wbx_acceptance"
    if not exe.exists():
        pytest.skip("wbx_acceptance not built (make -C oracle wbx-tests needs /root/reference)")
    # fp64: bitwise the reference; fp32: the hot path (the tracked window engine for the
    # energies the acceptance harness's ref_energy rule needs)
    env = dict(__import__("os").environ, WBX_BACKEND_PRECISION=precision)
    r = subprocess.run([str(exe), "/nonexistent-cli"], capture_output=True, text=True, timeout=1200, cwd=REF,
                       env=env)
    out = r.stdout
    for k in range(1, 9):
        assert f"PASS criterion {k}:" in out, out[-4000:]
