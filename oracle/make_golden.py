"""oracle/make_golden.py — TEST INFRASTRUCTURE ONLY.

Regenerates tests/golden/*.npz by running the UNMODIFIED reference (through
oracle/_ref/oracle_driver, which links oracle/_ref/libwaveblur_ref.so built from
/root/reference/proj/src by oracle/Makefile). Needs /root/reference, so it only runs
in the build container; the fixtures it writes are committed and travel.

    make -C oracle ref driver && python oracle/make_golden.py
"""
from __future__ import annotations

import json
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
DRIVER = HERE / "_ref" / "oracle_driver"
GOLDEN = HERE.parent / "tests" / "golden"

# name -> (driver args, which vectors to store)
CASES = {
    # BASELINE config C1: 256^2, db4 J=4, Gaussian sigma 5, K=3N dyadic,
    # noise 5e-3 seed 2024, lambda 1e-4, SPAI, 50 FISTA iterations.
    "c1_db4_256": (["--dims", "256", "256", "--family", "daubechies", "--order", "4", "--J", "4",
                    "--iters", "50"],
                   ["u0", "x0", "p", "x_final", "restored", "energies"]),
    # the reference acceptance fixture basis (acceptance.cpp:222-240): sym6 J=4
    "c1_sym6_256": (["--dims", "256", "256", "--family", "symmlet", "--order", "6", "--J", "4",
                     "--iters", "50"],
                    ["x_final", "energies"]),
    # BASELINE config C2 operator + scalars (vectors regenerated, checked by checksum)
    "c2_db4_1024": (["--dims", "1024", "1024", "--family", "daubechies", "--order", "4", "--J", "4",
                     "--iters", "100"],
                    ["energies"]),
    # small cases mirroring the reference's solver tests (test_solver.cpp:176-319)
    "s64_sym6_ista": (["--dims", "64", "64", "--family", "symmlet", "--order", "6", "--J", "3",
                       "--sigma", "3", "--K", "40000", "--noise", "5e-3", "--seed", "1",
                       "--precond", "identity", "--method", "ista", "--iters", "40"],
                      ["u0", "x0", "x_final", "restored", "energies"]),
    "s32_sym4_naive": (["--dims", "32", "32", "--family", "symmlet", "--order", "4", "--J", "2",
                        "--sigma", "2", "--K", "20000", "--mode", "uniform", "--noise", "0",
                        "--precond", "identity", "--iters", "25"],
                       ["u0", "x0", "x_final", "restored", "energies"]),
    "s64_sym6_spai": (["--dims", "64", "64", "--family", "symmlet", "--order", "6", "--J", "3",
                       "--sigma", "3", "--K", "60000", "--noise", "5e-3", "--seed", "3",
                       "--precond", "spai", "--iters", "200"],
                      ["u0", "x0", "p", "x_final", "restored", "energies"]),
    "s128_1d_sym6": (["--dims", "128", "--family", "symmlet", "--order", "6", "--J", "3",
                      "--sigma", "2", "--K", "3000", "--noise", "1e-3", "--seed", "7",
                      "--precond", "jacobi", "--iters", "60"],
                     ["u0", "x0", "p", "x_final", "restored", "energies"]),
    # ExactThetaOp (the FFT operator): kernel, apply / adjoint, tau, FISTA
    "exact_s64_sym6": (["--dims", "64", "64", "--family", "symmlet", "--order", "6", "--J", "3",
                        "--sigma", "3", "--K", "40000", "--noise", "5e-3", "--seed", "5",
                        "--precond", "identity", "--iters", "30", "--exact"],
                       ["u0", "x0", "psf", "exact_apply", "exact_adjoint", "exact_x_final", "exact_energies"]),
}


def run_case(name: str, args: list, keep: list) -> None:
    with tempfile.TemporaryDirectory() as td:
        out = Path(td)
        r = subprocess.run([str(DRIVER), "--out", str(out), *args], capture_output=True, text=True)
        if r.returncode != 0:
            raise SystemExit(f"{name}: driver failed ({r.returncode})\n{r.stderr}")
        meta = json.loads((out / "meta.json").read_text())
        assert meta["expand_ok"], name
        n = int(np.prod(meta["dims"]))
        arrays = {}
        gens = np.frombuffer((out / "gens.bin").read_bytes(),
                             dtype=np.dtype([("b", "<u4"), ("g", "<u4"), ("c", "<u8"), ("v", "<f8")]))
        arrays["gen_block"] = gens["b"].copy()
        arrays["gen_index"] = gens["g"].copy()
        arrays["gen_count"] = gens["c"].copy()
        arrays["gen_value"] = gens["v"].copy()
        for key in keep:
            arrays[key] = np.fromfile(out / f"{key}.bin", dtype="<f8")
        # checksums of the big vectors (for sizes whose vectors are not stored)
        for key in ["u0", "x0", "p", "x_final", "restored"]:
            f = out / f"{key}.bin"
            if f.exists():
                v = np.fromfile(f, dtype="<f8")
                assert v.size == n
                arrays[f"sum_{key}"] = np.array([v.sum(), np.sqrt((v * v).sum()), np.abs(v).max()])
        arrays["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
        GOLDEN.mkdir(parents=True, exist_ok=True)
        np.savez_compressed(GOLDEN / f"{name}.npz", **arrays)
        print(f"{name}: n={n} nnz={meta['nnz']} gens={meta['n_gens']} tau={meta.get('tau')} "
              f"-> {(GOLDEN / (name + '.npz')).stat().st_size / 1e3:.0f} kB", flush=True)


LADDER_SIGMAS = [2.5 + 5.0 * l / 7.0 for l in range(8)]


def make_ladder(size: int) -> None:
    """BASELINE configs C3/C4 (spatially varying blur, no reference implementation):
    the stationary Gaussian operators of an 8-level sigma ladder 2.5..7.5 px, each built
    and thresholded (K=3N, dyadic weights) by the reference itself. The spatially varying
    Theta_K is assembled from these by wbx_theta_varying (column-wise interpolation,
    SURVEY §8d)."""
    arrays = {"sigmas": np.array(LADDER_SIGMAS)}
    metas = []
    for l, s in enumerate(LADDER_SIGMAS):
        with tempfile.TemporaryDirectory() as td:
            out = Path(td)
            args = ["--dims", str(size), str(size), "--family", "daubechies", "--order", "4", "--J", "4",
                    "--sigma", repr(s), "--no-solve"]
            r = subprocess.run([str(DRIVER), "--out", str(out), *args], capture_output=True, text=True)
            if r.returncode != 0:
                raise SystemExit(f"ladder {size} level {l}: driver failed\n{r.stderr}")
            meta = json.loads((out / "meta.json").read_text())
            assert meta["expand_ok"]
            gens = np.frombuffer((out / "gens.bin").read_bytes(),
                                 dtype=np.dtype([("b", "<u4"), ("g", "<u4"), ("c", "<u8"), ("v", "<f8")]))
            for k, f in (("gen_block", "b"), ("gen_index", "g"), ("gen_count", "c"), ("gen_value", "v")):
                arrays[f"l{l}_{k}"] = gens[f].copy()
            metas.append(meta)
            print(f"ladder {size} sigma={s:.4f}: gens={meta['n_gens']} nnz={meta['nnz']}", flush=True)
    arrays["meta_json"] = np.frombuffer(json.dumps({"dims": [size, size], "family": "daubechies", "order": 4,
                                                    "J": 4, "levels": metas}).encode(), dtype=np.uint8)
    np.savez_compressed(GOLDEN / f"c3_ladder_{size}.npz", **arrays)


def main(names: list) -> None:
    if not DRIVER.exists():
        raise SystemExit("build the oracle first: make -C oracle ref driver")
    for name in names or list(CASES) + ["ladder256", "ladder1024"]:
        if name.startswith("ladder"):
            make_ladder(int(name[6:]))
        else:
            run_case(name, *CASES[name])


if __name__ == "__main__":
    main(sys.argv[1:])
