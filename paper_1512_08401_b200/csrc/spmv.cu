// Stand-alone SpMV entry points (y = Theta x, y = Theta^T x) over the compacted SELL-32
// layouts. Replaces spmv (theta.cpp:300-311), SparseThetaOp::apply/apply_adjoint
// (solver.cpp:11-17) and spmv_t (theta.cpp:344-356; the reference rebuilds the CSC per
// call, here the cached transpose layout is used — same in-row order, same result).
//
// Full-length vectors are gathered into the compacted column space, multiplied, and
// scattered back; empty rows produce 0.0 exactly as the reference's `double s = 0.0`.
#include "internal.hpp"
#include "sell.cuh"

namespace wbx {

namespace {

constexpr int kBlock = 256;

template <typename T>
__global__ void gather_kernel(const T* __restrict__ full, const uint32_t* __restrict__ idx, uint32_t m,
                              T* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = full[idx[i]];
}

template <typename T>
__global__ void scatter_kernel(const T* __restrict__ in, const uint32_t* __restrict__ idx, uint32_t m,
                               T* __restrict__ full) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) full[idx[i]] = in[i];
}

__global__ void sell_f64_kernel(SellView M, const double* __restrict__ x, double* __restrict__ y) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= M.xslices) return;
    const double v = sell_dot_f64_exact(M, warp, lane, x);
    const uint32_t r = warp * kWarp + lane;
    if (r < M.rows) y[r] = v;
}

__global__ void sell_f32_kernel(SellView M, const float* __restrict__ x, float* __restrict__ y) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= M.slices) return;
    float v = seg_partial<float, float>(M, warp, lane, x);
    const uint32_t r = seg_combine(M, warp, lane, v);
    if (r != kNoRow) y[r] = v;
}

inline unsigned blocks_for(uint64_t threads) {
    return static_cast<unsigned>((threads + kBlock - 1) / kBlock);
}

template <typename T>
DevBuf<T>& scratch_of(wbx_op* op, int which, uint64_t count) {
    DevBuf<T>& b = sizeof(T) == 8 ? reinterpret_cast<DevBuf<T>&>(op->scratch64[which])
                                  : reinterpret_cast<DevBuf<T>&>(op->scratch32[which]);
    if (b.n < count) b.alloc(count);
    return b;
}

template <typename T>
void full_spmv(wbx_op* op, int transpose, const T* x, T* y, cudaStream_t s) {
    const wbx_sell& M = transpose ? op->T : op->A;
    const uint32_t* in_idx = transpose ? op->R_glob.p : op->C_glob.p;   // gathered inputs
    const uint32_t* out_idx = transpose ? op->C_glob.p : op->R_glob.p;  // scattered outputs
    const uint32_t m_in = static_cast<uint32_t>(transpose ? op->nR : op->nC);
    const uint32_t m_out = static_cast<uint32_t>(M.rows);
    // compacted scratch cached on the operator (calls on one context are serialised)
    DevBuf<T>& xin = scratch_of<T>(op, 0, m_in > 0 ? m_in : 1);
    DevBuf<T>& yout = scratch_of<T>(op, 1, m_out > 0 ? m_out : 1);
    WBX_CUDA(cudaMemsetAsync(y, 0, op->n * sizeof(T), s));
    if (m_out > 0) {
        gather_kernel<T><<<blocks_for(m_in), kBlock, 0, s>>>(x, in_idx, m_in, xin.p);
        const SellView v = view_of(M);
        if constexpr (sizeof(T) == 8)
            sell_f64_kernel<<<blocks_for(uint64_t(v.xslices) * 32), kBlock, 0, s>>>(v, xin.p, yout.p);
        else
            sell_f32_kernel<<<blocks_for(uint64_t(v.slices) * 32), kBlock, 0, s>>>(v, xin.p, yout.p);
        scatter_kernel<T><<<blocks_for(m_out), kBlock, 0, s>>>(yout.p, out_idx, m_out, y);
        count_launch(op->ctx, 3);
        WBX_CUDA(cudaGetLastError());
    }
}

}  // namespace

void spmv_full_fp64(wbx_op* op, int transpose, const double* x_dev, double* y_dev, cudaStream_t s) {
    full_spmv<double>(op, transpose, x_dev, y_dev, s);
}

void spmv_full_fp32(wbx_op* op, int transpose, const float* x_dev, float* y_dev, cudaStream_t s) {
    if (!(op->A.seg_ok && op->T.seg_ok))
        fail(WBX_TOO_LARGE, "operator rows longer than 496 nonzeros: fp32 layout unavailable, use precision 64");
    full_spmv<float>(op, transpose, x_dev, y_dev, s);
}

// Compacted-space SpMV used by the kernel benchmark (bench.py --kernel spmv):
// y[R] = A x[C] with both vectors already compacted.
template <typename T>
void spmv_compact(wbx_ctx* ctx, const wbx_sell& M, const T* x, T* y, cudaStream_t s) {
    if (M.rows == 0) return;
    const SellView v = view_of(M);
    if constexpr (sizeof(T) == 8)
        sell_f64_kernel<<<blocks_for(uint64_t(v.xslices) * 32), kBlock, 0, s>>>(v, x, y);
    else
        sell_f32_kernel<<<blocks_for(uint64_t(v.slices) * 32), kBlock, 0, s>>>(v, x, y);
    count_launch(ctx);
    WBX_CUDA(cudaGetLastError());
}

template void spmv_compact<float>(wbx_ctx*, const wbx_sell&, const float*, float*, cudaStream_t);
template void spmv_compact<double>(wbx_ctx*, const wbx_sell&, const double*, double*, cudaStream_t);

}  // namespace wbx
