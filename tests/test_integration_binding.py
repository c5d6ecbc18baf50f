"""The reference-side binding of INTEGRATION.md (integration/wbx_backend.cpp) compiles against
the reference's own headers and this repo's C ABI (syntax check; build container only, where
/root/reference is mounted)."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_INC = Path("/root/reference/proj/include")


@pytest.mark.skipif(not REF_INC.exists() or shutil.which("g++") is None, reason="reference headers not mounted")
def test_backend_binding_compiles_against_reference_headers():
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{REF_INC}", f"-I{ROOT / 'include'}",
                        str(ROOT / "integration" / "wbx_backend.cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_backend_binding_matches_integration_md():
    md = (ROOT / "INTEGRATION.md").read_text()
    src = (ROOT / "integration" / "wbx_backend.cpp").read_text()
    assert src.strip() in md
