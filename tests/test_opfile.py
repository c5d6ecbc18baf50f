"""Operator files through the C ABI.

* WTHETA01 (theta.cpp:413-490): the reference's own file (tests/golden/s32_sym4_naive.wtheta,
  written by the unmodified reference's write_operator through oracle/_ref/oracle_driver
  --write-op) is read by wbx_read_operator into the reference's exact CSR, and
  wbx_write_operator reproduces its bytes; the reference's validation errors (CPU).
* WBXOP001, the device-ready operator cache: save -> load gives an operator whose solves are
  bitwise the freshly built one's, with P, tau and the solvers' window layouts restored (GPU)."""
from pathlib import Path

import numpy as np
import pytest

from paper_1512_08401_b200 import waveblur as W

REF_FILE = Path(__file__).resolve().parent / "golden" / "s32_sym4_naive.wtheta"


def test_reads_the_references_file_and_writes_its_bytes(golden, tmp_path):
    op = W.read_operator(str(REF_FILE))
    ref = golden("s32_sym4_naive").operator()
    assert op.n == ref.n == 1024
    assert np.array_equal(op.row_offsets, ref.row_offsets)
    assert np.array_equal(op.col_indices, ref.col_indices)
    assert np.array_equal(op.values, ref.values)
    assert op.family == W.FilterFamily.Symmlet and op.order == 4 and op.layout.J == 2
    out = tmp_path / "again.wtheta"
    W.write_operator(op, str(out))
    assert out.read_bytes() == REF_FILE.read_bytes()


@pytest.mark.parametrize("edit,match", [
    (lambda b: b"NOTTHETA" + b[8:], "not a WTHETA01"),
    (lambda b: b[:40], "truncated"),
    (lambda b: b[:8] + (3).to_bytes(4, "little") + b[12:], "bad dimension count"),
    (lambda b: b[:24] + (7).to_bytes(4, "little") + b[28:], "bad filter family"),
    (lambda b: b[:36] + (5).to_bytes(8, "little") + b[44:], "inconsistent row offsets"),
])
def test_validation_errors(tmp_path, edit, match):
    raw = REF_FILE.read_bytes()
    bad = tmp_path / "bad.wtheta"
    bad.write_bytes(edit(raw))
    with pytest.raises(W.IoError, match=match):
        W.read_operator(str(bad))
    with pytest.raises(W.IoError, match="cannot open"):
        W.read_operator(str(tmp_path / "missing.wtheta"))


@pytest.mark.gpu
def test_device_cache_roundtrip(golden, tmp_path):
    g = golden("c1_db4_256")
    op = g.operator()
    ctx = W.Context(0)
    basis = W.make_basis(W.FilterFamily.Daubechies, 4, (256, 256), 4)
    P = W.spai(op, ctx)
    w = g.weights()
    cfg = W.SolverConfig(max_iters=50, track_energy=False)
    d = W.Deblurrer(op, basis, P, w, 1e-4, cfg, ctx)   # builds the window layouts on the operator
    ref, rep = d.deblur(g["u0"], clamp=True)
    path = tmp_path / "c1.wbxop"
    W.save_device_operator(op, str(path), P, rep.tau, ctx)
    ctx2 = W.Context(0)
    op2, P2, tau2 = W.load_device_operator(str(path), ctx2, op.layout)
    assert np.array_equal(op2.row_offsets, op.row_offsets) and np.array_equal(op2.values, op.values)
    assert np.array_equal(P2.p, P.p) and tau2 == rep.tau
    d2 = W.Deblurrer(op2, basis, P2, w, 1e-4, cfg, ctx2)
    out, rep2 = d2.deblur(g["u0"], clamp=True)
    assert np.array_equal(out, ref) and rep2.tau == rep.tau
    assert d2.kernels() == d.kernels()
    # spmv on the loaded layouts: bitwise the fresh operator's (fp64 reference order)
    x = np.random.default_rng(2).standard_normal(op.n)
    assert np.array_equal(W.spmv(op2, x, ctx2), W.spmv(op, x, ctx))
    bad = tmp_path / "bad.wbxop"
    bad.write_bytes(path.read_bytes()[:1000])
    with pytest.raises(W.IoError):
        W.load_device_operator(str(bad), ctx2)
