"""Copy integration/wbx_backend.cpp into the ```cpp block of INTEGRATION.md §2
(tests/test_integration_binding.py checks the two are identical)."""
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
md = (ROOT / "INTEGRATION.md").read_text()
src = (ROOT / "integration" / "wbx_backend.cpp").read_text().strip()
a = md.index("```cpp\n") + len("```cpp\n")
b = md.index("\n```\n", a)
(ROOT / "INTEGRATION.md").write_text(md[:a] + src + md[b:])
