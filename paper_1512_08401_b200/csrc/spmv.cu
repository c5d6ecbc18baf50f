// Stand-alone SpMV entry points (y = Theta x, y = Theta^T x) over the compacted SELL-32
// layouts. Replaces spmv (theta.cpp:300-311), SparseThetaOp::apply/apply_adjoint
// (solver.cpp:11-17) and spmv_t (theta.cpp:344-356; the reference rebuilds the CSC per
// call, here the cached transpose layout is used — same in-row order, same result).
//
// Full-length vectors are gathered into the compacted column space, multiplied, and
// scattered back; empty rows produce 0.0 exactly as the reference's `double s = 0.0`.
#include <cstdlib>
#include <cstring>

#include "internal.hpp"
#include "sell.cuh"
#include "stream.cuh"

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

// The register-staged kernel in parts of H pairs per lane: fewer live registers, so more
// warps per SM hide the record -> gather chain (H = 4: 40 registers, 48 warps/SM; 4096^2
// forward 100 us vs 118 us for all 8 pairs at once). Same fma order as seg_partial.
template <int H, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) sell_f32_part_kernel(SellView M, const float* __restrict__ x,
                                                                     float* __restrict__ y) {
    const uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= M.slices) return;
    const uint4* p = M.pk + M.slice_ptr[s] + lane;
    const int np = static_cast<int>(M.slice_np[s] & 0xffu);
    const uint64_t pol = l2_keep_policy();
    float acc = 0.f;
#pragma unroll
    for (int h = 0; h < 8; h += H) {
        if (h < np) {
            uint4 e[H];
#pragma unroll
            for (int j = 0; j < H; ++j) e[j] = h + j < np ? ld_stream(p + (h + j) * kWarp, pol) : make_uint4(0, 0, 0, 0);
            float g[2 * H];
#pragma unroll
            for (int j = 0; j < H; ++j) {
                g[2 * j] = h + j < np ? x[e[j].y] : 0.f;
                g[2 * j + 1] = h + j < np ? x[e[j].w] : 0.f;
            }
#pragma unroll
            for (int j = 0; j < H; ++j) {
                if (h + j < np) {
                    acc = fmaf(__uint_as_float(e[j].x), g[2 * j], acc);
                    acc = fmaf(__uint_as_float(e[j].z), g[2 * j + 1], acc);
                }
            }
        }
    }
    const uint32_t r = seg_combine(M, s, lane, acc);
    if (r != kNoRow) y[r] = acc;
}

// Row-per-lane fp32 SpMV (the default standalone kernel): slice s = the 32 consecutive
// sorted rows 32s..32s+31, one per lane; the lane walks its row in element order in parts
// of H {val, col, val, col} pairs (16-B loads, 512 B per warp instruction), then the odd
// last element. Rows of a slice have ~equal length (the compacted rows are sorted by
// length), so the stream carries no segment padding and no per-lane row word: 8 B per
// nonzero plus 8 B per 32 rows. The operator stream is loaded EVICT_FIRST (read once;
// it must not push x out of L2), and each warp issues a bulk L2 prefetch of the stream
// window PF bytes ahead of its own slice (the ranges tile the stream, so every byte is
// prefetched once and the prefetch front runs PF bytes ahead of the compute front):
// HBM requests are in flight without holding registers or shared memory.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int H, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) sell_row_kernel(SellView M, const float* __restrict__ x,
                                                             float* __restrict__ y, uint64_t pf_u4) {
    const uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= M.xslices) return;
    const uint2 meta = M.rslice[s];
    const uint32_t L = meta.y, np = L >> 1;
    if (pf_u4 != 0 && lane == 0) {
        const uint64_t a = uint64_t(meta.x) + pf_u4;
        uint64_t b = uint64_t(meta.x) + np * 32u + (L & 1u) * 16u + pf_u4;
        if (b > M.rpk_u4) b = M.rpk_u4;
        if (a < b) prefetch_l2_bulk(M.rpk + a, static_cast<uint32_t>((b - a) * 16u));
    }
    const uint4* p = M.rpk + meta.x + lane;
    const uint64_t pol = l2_evict_first_policy();
    float acc = 0.f;
    for (uint32_t h = 0; h < np; h += H) {
        uint4 e[H];
#pragma unroll
        for (int j = 0; j < H; ++j) e[j] = h + j < np ? ld_stream(p + (h + j) * kWarp, pol) : make_uint4(0, 0, 0, 0);
        float g[2 * H];
#pragma unroll
        for (int j = 0; j < H; ++j) {
            g[2 * j] = h + j < np ? x[e[j].y] : 0.f;
            g[2 * j + 1] = h + j < np ? x[e[j].w] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < H; ++j) {
            if (h + j < np) {
                acc = fmaf(__uint_as_float(e[j].x), g[2 * j], acc);
                acc = fmaf(__uint_as_float(e[j].z), g[2 * j + 1], acc);
            }
        }
    }
    if (L & 1u) {
        const uint2 t = ld_stream(reinterpret_cast<const uint2*>(M.rpk + meta.x + np * 32u) + lane, pol);
        acc = fmaf(__uint_as_float(t.x), x[t.y], acc);
    }
    const uint32_t r = s * kWarp + lane;
    if (r < M.rows) y[r] = acc;
}

// fp32 SELL SpMV with the operator stream staged by the TMA engine. Each warp walks the
// slices gw, gw + TW, ... (TW = warps in the grid); lane 0 keeps the warp's next
// slice records ([lane_info 32 x u32][np x 32 pairs]) in flight as 1-D bulk copies into a
// shared-memory ring, so the bytes in flight per SM are set by shared memory, not by
// registers. Measured slower than the register-staged kernels (~55-65 % of HBM at
// 4096^2): the limiter is each warp's dependent record -> x-gather round trip, not the
// bytes in flight, and the ring's shared memory caps the warps per SM at 12-24. Same loads,
// gathers and fma order per lane as seg_partial/seg_combine: bitwise equal results.
constexpr unsigned kRecU4Max = 8u + kSlotBytes / 16u;     // uint4 per slot
constexpr unsigned kSlotStride = kRecU4Max * 16u + 8u + 4u; // slot + mbarrier + np word

__device__ __forceinline__ uint64_t l2_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// NS slices per warp iteration (their x gathers issued together), KS ring slots per warp
// (NS being consumed, KS - NS in flight). Per-slice arithmetic is that of seg_partial/seg_combine.
template <int NS, int KS, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) sell_f32_tma_kernel(SellView M, const float* __restrict__ x,
                                                                   float* __restrict__ y) {
    constexpr int kS = KS;
    static_assert(KS >= NS, "ring smaller than a group");
    extern __shared__ __align__(128) unsigned char sm[];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint4* ring = reinterpret_cast<uint4*>(sm) + size_t(wib) * kS * kRecU4Max;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + size_t(WARPS) * kS * kRecU4Max * 16u) + wib * kS;
    uint32_t* snp = reinterpret_cast<uint32_t*>(sm + size_t(WARPS) * kS * (kRecU4Max * 16u + 8u)) + wib * kS;
    const uint64_t TW = uint64_t(gridDim.x) * WARPS;
    const uint64_t gw = uint64_t(blockIdx.x) * WARPS + wib;
    const uint64_t pol = l2_first_policy();
    auto issue = [&](uint64_t s, int slot) {  // lane 0
        const uint64_t o0 = M.rec_off[s], o1 = M.rec_off[s + 1];
        const unsigned bytes = static_cast<unsigned>((o1 - o0) * 16u);
        snp[slot] = M.slice_np[s];
        mbar_expect_tx(bars + slot, bytes);
        bulk_g2s(ring + size_t(slot) * kRecU4Max, M.rec + o0, bytes, bars + slot, pol);
    };
    if (lane == 0) {
        for (int i = 0; i < kS; ++i) mbar_init(bars + i, 1);
        mbar_fence_init();
        for (int i = 0; i < kS; ++i) {
            const uint64_t s = gw + uint64_t(i) * TW;
            if (s < M.slices) issue(s, i);
        }
    }
    __syncwarp();
    for (uint64_t k = 0;; k += NS) {
        if (gw + k * TW >= M.slices) break;
        float g[NS][16];
        uint32_t word[NS], info[NS];
        const uint4* r[NS];
#pragma unroll
        for (int t = 0; t < NS; ++t) {
            const uint64_t s = gw + (k + t) * TW;
            const int slot = static_cast<int>((k + t) % kS);
            r[t] = ring + size_t(slot) * kRecU4Max;
            word[t] = 0;
            info[t] = kNoRow;
            if (s < M.slices) {
                mbar_wait(bars + slot, ((k + t) / kS) & 1u);
                word[t] = snp[slot];
                info[t] = reinterpret_cast<const uint32_t*>(r[t])[lane];
            }
            const uint32_t np = word[t] & 0xffu;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j < static_cast<int>(np)) {
                    const uint4 e = r[t][8 + j * kWarp + lane];
                    g[t][2 * j] = x[e.y];
                    g[t][2 * j + 1] = x[e.w];
                } else {
                    g[t][2 * j] = 0.f;
                    g[t][2 * j + 1] = 0.f;
                }
            }
        }
        float acc[NS];
#pragma unroll
        for (int t = 0; t < NS; ++t) {
            const uint32_t np = word[t] & 0xffu;
            acc[t] = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j < static_cast<int>(np)) {
                    const uint4 e = r[t][8 + j * kWarp + lane];
                    acc[t] = fmaf(__uint_as_float(e.x), g[t][2 * j], acc[t]);
                    acc[t] = fmaf(__uint_as_float(e.z), g[t][2 * j + 1], acc[t]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) {  // the NS slots are consumed: refill them kS slices ahead
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
            for (int t = 0; t < NS; ++t) {
                const uint64_t sn = gw + (k + t + kS) * TW;
                if (sn < M.slices) issue(sn, static_cast<int>((k + t) % kS));
            }
        }
#pragma unroll
        for (int t = 0; t < NS; ++t) {
            const uint32_t m = word[t] >> 8;
            const uint32_t nseg = info[t] == kNoRow ? 1u : (info[t] >> 27);
            const uint32_t maxseg = __reduce_max_sync(0xffffffffu, nseg);
            float v = acc[t];
            for (uint32_t j = 1; j < maxseg; ++j) {
                const float u = __shfl_down_sync(0xffffffffu, v, j * m);
                if (j < nseg) v += u;
            }
            if (info[t] != kNoRow) y[info[t] & kRowMask] = v;
        }
    }
}

// WBX_SPMV: row (default, sell_row_kernel<4>: row-per-lane layout, 4 pairs per step, 32
// registers, 64 warps/SM) | row2 | row8 (2 / 8 pairs per step) | quarter | half | reg (segmented
// layout: sell_f32_part_kernel<2>, <4>, sell_f32_kernel) | tma1 | tma2 | tma3 (TMA-staged
// segmented variants). 4096^2 fp32 forward, L2 flushed: row 75.8 us (0.84 of HBM), row2 77.8,
// quarter 97, half 100, reg 118, tma1 137, tma2 158, tma3 132 us (tools/spmv_sweep.py,
// profiles/r02_spmv_roofline.md, profiles/r01_spmv_roofline.md)
int spmv_mode() {
    static const int mode = [] {
        const char* e = std::getenv("WBX_SPMV");
        if (e && std::strcmp(e, "tma1") == 0) return 1;
        if (e && std::strcmp(e, "tma2") == 0) return 2;
        if (e && std::strcmp(e, "tma3") == 0) return 3;
        if (e && std::strcmp(e, "reg") == 0) return 0;
        if (e && std::strcmp(e, "half") == 0) return 4;
        if (e && std::strcmp(e, "quarter") == 0) return 5;
        if (e && std::strcmp(e, "row2") == 0) return 6;
        if (e && std::strcmp(e, "row8") == 0) return 8;
        return 7;
    }();
    return mode;
}

template <int NS, int KS, int WARPS, int MINB>
void launch_tma(wbx_ctx* ctx, const SellView& v, const float* x, float* y, cudaStream_t s) {
    constexpr size_t smem = size_t(WARPS) * KS * kSlotStride;
    static bool attr = false;
    if (!attr) {
        WBX_CUDA(cudaFuncSetAttribute(sell_f32_tma_kernel<NS, KS, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        attr = true;
    }
    const uint64_t want = (uint64_t(v.slices) + WARPS - 1) / WARPS;
    const uint64_t cap = uint64_t(ctx->num_sms > 0 ? ctx->num_sms : 148) * MINB;
    const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
    sell_f32_tma_kernel<NS, KS, WARPS><<<grid, WARPS * 32, smem, s>>>(v, x, y);
}

// L2 prefetch distance of the row kernel (bytes ahead in the operator stream; WBX_SPMV_PF,
// 0 disables)
long long g_spmv_pf_bytes = -1;  // wbx_diag_set_spmv_pf (sweeps); -1: WBX_SPMV_PF or the default

uint64_t spmv_pf_u4() {
    static const uint64_t pf = [] {
        const char* e = std::getenv("WBX_SPMV_PF");
        const long long b = e ? std::atoll(e) : 0ll;  // measured: the prefetch costs 13-20 % (r02 sweep)
        return static_cast<uint64_t>(b > 0 ? b : 0) / 16u;
    }();
    return g_spmv_pf_bytes >= 0 ? static_cast<uint64_t>(g_spmv_pf_bytes) / 16u : pf;
}

void launch_sell_f32(wbx_ctx* ctx, const SellView& v, const float* x, float* y, cudaStream_t s, int mode) {
    if (mode >= 6) {
        const unsigned rb = static_cast<unsigned>((uint64_t(v.xslices) * 32 + kBlock - 1) / kBlock);
        if (mode == 6)
            sell_row_kernel<2, 8><<<rb, kBlock, 0, s>>>(v, x, y, spmv_pf_u4());
        else if (mode == 7)
            sell_row_kernel<4, 8><<<rb, kBlock, 0, s>>>(v, x, y, spmv_pf_u4());
        else
            sell_row_kernel<8, 4><<<rb, kBlock, 0, s>>>(v, x, y, spmv_pf_u4());
        return;
    }
    const unsigned blocks = static_cast<unsigned>((uint64_t(v.slices) * 32 + kBlock - 1) / kBlock);
    if (mode == 4)
        sell_f32_part_kernel<4, 6><<<blocks, kBlock, 0, s>>>(v, x, y);
    else if (mode == 5)
        sell_f32_part_kernel<2, 8><<<blocks, kBlock, 0, s>>>(v, x, y);
    else if (mode == 3)
        launch_tma<1, 2, 12, 2>(ctx, v, x, y, s);  // 24 warps/SM, 2 slots each: 2 x 102 KB smem
    else if (mode == 2)
        launch_tma<2, 4, 4, 3>(ctx, v, x, y, s);   // 12 warps/SM, 2 slices per step: 3 x 68 KB
    else if (mode == 1)
        launch_tma<1, 3, 8, 2>(ctx, v, x, y, s);   // 16 warps/SM, 3 slots each: 2 x 102 KB
    else
        sell_f32_kernel<<<static_cast<unsigned>((uint64_t(v.slices) * 32 + kBlock - 1) / kBlock), kBlock, 0, s>>>(v, x, y);
}

inline unsigned blocks_for(uint64_t threads) {
    return static_cast<unsigned>((threads + kBlock - 1) / kBlock);
}

// compacted scratch of the CALLING context (calls on one context are serialised; two
// contexts sharing an operator never share scratch)
template <typename T>
DevBuf<T>& scratch_of(wbx_ctx* ctx, int which, uint64_t count) {
    DevBuf<T>& b = sizeof(T) == 8 ? reinterpret_cast<DevBuf<T>&>(ctx->scratch64[which])
                                  : reinterpret_cast<DevBuf<T>&>(ctx->scratch32[which]);
    if (b.n < count) b.alloc(count);
    return b;
}

template <typename T>
void full_spmv(wbx_ctx* ctx, const wbx_op* op, int transpose, const T* x, T* y, cudaStream_t s) {
    const wbx_sell& M = transpose ? op->T : op->A;
    const uint32_t* in_idx = transpose ? op->R_glob.p : op->C_glob.p;   // gathered inputs
    const uint32_t* out_idx = transpose ? op->C_glob.p : op->R_glob.p;  // scattered outputs
    const uint32_t m_in = static_cast<uint32_t>(transpose ? op->nR : op->nC);
    const uint32_t m_out = static_cast<uint32_t>(M.rows);
    DevBuf<T>& xin = scratch_of<T>(ctx, 0, m_in > 0 ? m_in : 1);
    DevBuf<T>& yout = scratch_of<T>(ctx, 1, m_out > 0 ? m_out : 1);
    WBX_CUDA(cudaMemsetAsync(y, 0, op->n * sizeof(T), s));
    if (m_out > 0) {
        gather_kernel<T><<<blocks_for(m_in), kBlock, 0, s>>>(x, in_idx, m_in, xin.p);
        const SellView v = view_of(M);
        if constexpr (sizeof(T) == 8)
            sell_f64_kernel<<<blocks_for(uint64_t(v.xslices) * 32), kBlock, 0, s>>>(v, xin.p, yout.p);
        else
            launch_sell_f32(ctx, v, xin.p, yout.p, s, spmv_mode());
        scatter_kernel<T><<<blocks_for(m_out), kBlock, 0, s>>>(yout.p, out_idx, m_out, y);
        count_launch(ctx, 3);
        WBX_CUDA(cudaGetLastError());
    }
}

}  // namespace

void set_spmv_pf_bytes(long long b) { g_spmv_pf_bytes = b; }

void spmv_full_fp64(wbx_ctx* ctx, const wbx_op* op, int transpose, const double* x_dev, double* y_dev) {
    full_spmv<double>(ctx, op, transpose, x_dev, y_dev, ctx->stream);
}

void spmv_full_fp32(wbx_ctx* ctx, const wbx_op* op, int transpose, const float* x_dev, float* y_dev) {
    if (!(op->A.seg_ok && op->T.seg_ok))
        fail(WBX_TOO_LARGE, "operator rows longer than 496 nonzeros: fp32 layout unavailable, use precision 64");
    full_spmv<float>(ctx, op, transpose, x_dev, y_dev, ctx->stream);
}

// Compacted-space SpMV used by the kernel benchmark (bench.py --kernel spmv):
// y[R] = A x[C] with both vectors already compacted.
template <typename T>
void spmv_compact(wbx_ctx* ctx, const wbx_sell& M, const T* x, T* y, cudaStream_t s, int mode) {
    if (M.rows == 0) return;
    const SellView v = view_of(M);
    if constexpr (sizeof(T) == 8)
        sell_f64_kernel<<<blocks_for(uint64_t(v.xslices) * 32), kBlock, 0, s>>>(v, x, y);
    else
        launch_sell_f32(ctx, v, x, y, s, mode < 0 ? spmv_mode() : mode);
    count_launch(ctx);
    WBX_CUDA(cudaGetLastError());
}

template void spmv_compact<float>(wbx_ctx*, const wbx_sell&, const float*, float*, cudaStream_t, int);
template void spmv_compact<double>(wbx_ctx*, const wbx_sell&, const double*, double*, cudaStream_t, int);

}  // namespace wbx
