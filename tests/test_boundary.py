"""The drop-in boundary on CPU: libwbx.so loads, exports every symbol include/wbx.h
declares, and its host-only entry points (filters, layout, weights, the generator-list
expansion, argument validation) match the oracle / reference conventions."""
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_08401_b200 import _native as N
from paper_1512_08401_b200 import waveblur as W

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "wbx.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(wbx_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(N.lib, s), f"libwbx.so does not export {s}"
    assert set(syms) == set(N.SIGNATURES), "ctypes signature table out of sync with include/wbx.h"
    assert N.lib.wbx_abi_version() == 1


@pytest.mark.parametrize("fam,order", [(0, 1), (1, 2), (1, 4), (1, 10), (2, 4), (2, 6), (2, 8)])
def test_filters_bitwise_equal_to_oracle(fam, order):
    f = W.make_filters(W.FilterFamily(fam), order)
    lo, hi = O.filters(fam, order)
    assert np.array_equal(f.lowpass, lo) and np.array_equal(f.highpass, hi)


def test_filter_names_and_errors():
    # test_wavelet.cpp:68-76
    assert W.make_filters("sym6").length() == 12
    assert W.make_filters("symmlet6").length() == 12
    assert W.make_filters("db4").length() == 8
    for bad in [("nonsense",), (W.FilterFamily.Daubechies, 11), (W.FilterFamily.Daubechies, 1),
                (W.FilterFamily.Symmlet, 3)]:
        with pytest.raises(W.UnsupportedFilter):
            W.make_filters(*bad)


def test_layout_partitions_and_shapes():
    # test_wavelet.cpp:79-102
    L = W.make_layout((32, 64), 3)
    assert L.total() == 32 * 64
    covered = 0
    for b in L.bands:
        assert b.offset == covered
        covered += b.count()
        if b.orientation == 0:
            assert b.level == L.J
    assert L.find(3, 0).shape == (4, 8)
    assert L.find(1, 3).shape == (16, 32)
    for bad in [((48,), 2), ((16,), 5)]:
        with pytest.raises(W.ShapeMismatch):
            W.make_layout(*bad)
    with pytest.raises(W.ShapeMismatch):
        W.make_layout((), 1)


def test_scale_weights_follow_levels():
    # test_solver.cpp:321-328
    L = W.make_layout((32, 32), 3)
    w = W.scale_weights(L)
    for b in L.bands:
        expect = 3.0 if b.orientation == 0 else float(b.level)
        assert np.all(w[b.offset:b.offset + b.count()] == expect)


def test_generator_expansion_structure(golden):
    g = golden("c2_db4_1024")
    op = g.operator()
    assert op.nnz() == g.meta["nnz"] == 3 * g.n
    ro = op.row_offsets.astype(np.int64)
    assert ro[0] == 0 and ro[-1] == op.nnz() and np.all(np.diff(ro) >= 0)
    rows = np.repeat(np.arange(op.n), np.diff(ro))
    same = rows[1:] == rows[:-1]
    assert np.all(op.col_indices[1:][same] > op.col_indices[:-1][same])
    # SURVEY §0.3 structure at 1024^2, K=3N: 14.8 % nonempty rows, 4.69 % nonempty columns
    nz_rows = np.count_nonzero(np.diff(ro))
    nz_cols = np.unique(op.col_indices).size
    assert abs(nz_rows / op.n - 0.1484) < 0.002
    assert nz_cols == 49152


def test_generator_expansion_rejects_bad_input():
    gl = W.GeneratorList((16, 16), 2, W.FilterFamily.Haar, 1, np.array([999], np.uint32),
                         np.array([0], np.uint32), np.array([1], np.uint64), np.array([1.0]))
    with pytest.raises(W.BandNotFound):
        W.theta_from_generators(gl)


def test_wtheta01_roundtrip(tmp_path, golden):
    # test_io.cpp:102-129
    op = golden("s64_sym6_spai").operator()
    p = tmp_path / "op.wtheta"
    W.write_operator(op, str(p))
    back = W.read_operator(str(p))
    assert back.n == op.n and np.array_equal(back.row_offsets, op.row_offsets)
    assert np.array_equal(back.col_indices, op.col_indices) and np.array_equal(back.values, op.values)
    raw = bytearray(p.read_bytes())
    raw[0:8] = b"NOTTHETA"
    (tmp_path / "bad").write_bytes(bytes(raw))
    with pytest.raises(W.IoError):
        W.read_operator(str(tmp_path / "bad"))
    (tmp_path / "short").write_bytes(bytes(p.read_bytes()[:40]))
    with pytest.raises(W.IoError):
        W.read_operator(str(tmp_path / "short"))


def test_host_transpose_matches_oracle(golden):
    op = golden("s64_sym6_spai").operator()
    t = W.transpose(op)
    ot = O.Csr.of(op).transpose()
    assert np.array_equal(t.row_offsets, ot.ro) and np.array_equal(t.col_indices, ot.ci)
    assert np.array_equal(t.values, ot.va)
