"""The stencil engine's plan (csrc/stencil_plan.cu), executed on the host (CPU, no GPU).

The plan turns the reference's kept generator groups (theta.cpp:236-275) into per-tile
windows and affine tap lists; wbx_diag_stencil_apply_host runs it with the device kernel's
windows, offsets and summation order. Its products must be the CSR's (the operator the
reference assembles from the same groups, theta.cpp:180-201) with the values in fp32."""
import numpy as np
import pytest

from paper_1512_08401_b200 import _native as N
from paper_1512_08401_b200 import waveblur as W

CASES = ["c1_db4_256", "c1_sym6_256", "c2_db4_1024", "exact_s64_sym6", "s32_sym4_naive", "s64_sym6_spai"]


def stencil_apply(gl, phase, G, x):
    dims = np.array(gl.dims, dtype=np.uint64)
    y = np.full(x.size, np.nan)
    W._check(N.lib.wbx_diag_stencil_apply_host(len(gl.dims), W._u64ptr(dims), gl.J, gl.blocks.size,
                                                 W._u32ptr(gl.blocks), W._u32ptr(gl.gen_index),
                                                 W._u64ptr(gl.counts), W._dptr(gl.values), phase, G,
                                                 W._dptr(np.ascontiguousarray(x)), W._dptr(y)))
    return y


def csr_products(op, x):
    """Theta x and Theta^T x with the values rounded to fp32 (the engine's records), in double."""
    v = op.values.astype(np.float32).astype(np.float64)
    rows = np.repeat(np.arange(op.n), np.diff(op.row_offsets.astype(np.int64)))
    cols = op.col_indices.astype(np.int64)
    ax = np.zeros(op.n)
    np.add.at(ax, rows, v * x[cols])
    atx = np.zeros(op.n)
    np.add.at(atx, cols, v * x[rows])
    return ax, atx, np.unique(rows), np.unique(cols)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("G", [148, 296])
def test_stencil_plan_matches_csr(golden, name, G):
    g = golden(name)
    gl = g.generator_list()
    op = W.theta_from_generators(gl)
    x = np.random.default_rng(7).standard_normal(op.n)
    ax, atx, rows, cols = csr_products(op, x)
    ya = stencil_apply(gl, 0, G, x)
    yt = stencil_apply(gl, 1, G, x)
    # every nonzero row (column) lies in an output band of phase A (T); the rest stays untouched
    assert np.isfinite(ya[rows]).all() and np.isfinite(yt[cols]).all()
    ma, mt = np.isfinite(ya), np.isfinite(yt)
    assert np.all(ax[~ma] == 0) and np.all(atx[~mt] == 0)
    scale_a = np.abs(ax).max()
    scale_t = np.abs(atx).max()
    assert np.abs(ya[ma] - ax[ma]).max() <= 1e-12 * scale_a
    assert np.abs(yt[mt] - atx[mt]).max() <= 1e-12 * scale_t


def test_stencil_plan_rejects_1d(golden):
    gl = golden("s128_1d_sym6").generator_list()
    x = np.zeros(128)
    with pytest.raises(W.BadSpec, match="2-D"):
        stencil_apply(gl, 0, 148, x)
