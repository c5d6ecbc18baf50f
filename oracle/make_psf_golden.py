"""oracle/make_psf_golden.py — TEST INFRASTRUCTURE ONLY.

Writes tests/golden/psf_cases.npz from the UNMODIFIED reference (oracle/_ref/psf_driver,
linked against oracle/_ref/libwaveblur_ref.so built from /root/reference): generate_psf for
every PsfSpec kind (operators.cpp:98-318), convolve / apply_adjoint / add_noise / degrade of
the synthetic scene (operators.cpp:320-387). Needs /root/reference (build container only).

    make -C oracle ref psf-driver && python oracle/make_psf_golden.py
"""
import hashlib
import json
import subprocess
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT = HERE.parent / "tests" / "golden" / "psf_cases.npz"
BIG = 1 << 16  # kernels with more pixels are stored as sha256 of their bytes only

with tempfile.TemporaryDirectory() as td:
    subprocess.run([str(HERE / "_ref" / "psf_driver"), td], check=True)
    arrays, index = {}, []
    for line in (Path(td) / "index.txt").read_text().splitlines():
        name, spec, *dims = line.split()
        dims = [int(d) for d in dims]
        k = np.fromfile(Path(td) / f"{name}.bin", dtype="<f8")
        entry = {"name": name, "spec": spec, "dims": dims}
        if k.size > BIG:
            entry["sha256"] = hashlib.sha256(k.tobytes()).hexdigest()
        else:
            arrays[f"k_{name}"] = k
        index.append(entry)
    for key in ("scene64", "conv64", "adj64", "degrade64", "noise64"):
        arrays[key] = np.fromfile(Path(td) / f"{key}.bin", dtype="<f8")
    arrays["index_json"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
print(OUT, OUT.stat().st_size)
