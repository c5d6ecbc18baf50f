"""bench.py's multi-GPU launch path on CPU: `--gpus 2` outside torchrun re-executes itself
under torch.distributed.run (127.0.0.1 rendezvous). The reference arm needs no GPU: rank 0
times the reference's own CPU deblur and prints one JSON line with n_gpus 2 and the same
config object the GPU arm emits; rank 1 exits without work. The arm must not load libwbx.so."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
DRIVER = ROOT / "oracle" / "_ref" / "oracle_driver"


@pytest.mark.skipif(not DRIVER.exists(), reason="oracle/_ref/oracle_driver not built (needs /root/reference)")
def test_reference_arm_spawns_two_ranks():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "0", "--no-single-thread"], capture_output=True, text=True, timeout=600,
                       cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["cpu_baseline"]["kind"] == "reference" and line["value"] > 0
    sys.path.insert(0, str(ROOT))
    import bench
    assert line["config"] == bench.bench_config(2)


def test_reference_arm_imports_no_native_code():
    code = ("import sys, runpy; sys.argv=['bench.py']; g = runpy.run_path('bench.py', run_name='bench'); "
            "g['bench_config'](1); import numpy; "
            "print('libwbx' in open('/proc/self/maps').read(), any(m.startswith('paper_1512_08401_b200.') "
            "for m in sys.modules))")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=str(ROOT), timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.split() == ["False", "False"], r.stdout
