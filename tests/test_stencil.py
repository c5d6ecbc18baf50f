"""Circulant-compressed Theta_K applied as a stencil SpMV, against the CSR
SpMV of the same operator (which is bitwise the reference's): fp64 within summation-order
rounding, fp32 within fp32 rounding; forward and adjoint; 1-D and 2-D; naive and dyadic
thresholds; C2 size."""
import numpy as np
import pytest

from paper_1512_08401_b200 import _native as N
from paper_1512_08401_b200 import waveblur as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["s128_1d_sym6", "s32_sym4_naive", "s64_sym6_spai", "c1_db4_256", "c2_db4_1024"])
def test_stencil_matches_csr(golden, name):
    import torch
    g = golden(name)
    op = g.operator()
    gl = g.generator_list()
    st = W.StencilOperator(gl)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(op.n)
    dev = torch.device("cuda", 0)
    for transpose in (False, True):
        ref = W.spmv_t(op, x) if transpose else W.spmv(op, x)
        xd = torch.from_numpy(x).to(dev)
        yd = torch.empty_like(xd)
        torch.cuda.synchronize()
        st.spmv_dev(xd.data_ptr(), yd.data_ptr(), transpose, N.WBX_FP64)
        W.default_context().synchronize()
        y = yd.cpu().numpy()
        scale = np.abs(ref).max()
        assert np.abs(y - ref).max() <= 1e-13 * scale, (name, transpose)
        x32 = xd.float()
        y32 = torch.empty_like(x32)
        torch.cuda.synchronize()
        st.spmv_dev(x32.data_ptr(), y32.data_ptr(), transpose, N.WBX_FP32)
        W.default_context().synchronize()
        assert np.abs(y32.cpu().numpy() - ref).max() <= 1e-5 * scale, (name, transpose)
