// Sliced-ELL row dot products over the two device layouts of an operator.
//
// * Segmented fp32 layout (the hot path): every row is cut into segments of at most
//   kSegElems = 16 nonzeros; one lane owns one segment and a row's segments sit in
//   consecutive lanes of one 32-lane slice. A lane issues all of its (<= 8) 16-byte
//   {val,col,val,col} loads back to back, then the (<= 16) gathers, so a warp's
//   dependency chain is two memory round trips regardless of row length (rows reach 99
//   nonzeros in Theta and 137 in Theta^T at 1024^2). Segment partials are combined by
//   warp shuffles into the row's head lane in a fixed order (deterministic).
// * Exact fp64 layout: one lane per row, the row summed SEQUENTIALLY in element order —
//   the reference's in-row order (theta.cpp:306-308) with no FMA contraction — so it
//   reproduces the reference's spmv bit for bit.
#pragma once

#include "device_util.cuh"

namespace wbx {

struct SellView {
    // exact fp64
    const uint64_t* xslice_ptr;
    const uint32_t* xslice_len;
    const double* v64;
    const uint32_t* col;
    const uint32_t* row_len;
    // segmented fp32
    const uint64_t* slice_ptr;
    const uint32_t* slice_np;
    const uint4* pk;
    const uint32_t* lane_info;
    const uint4* rec;          // slice records [lane_info x32][pairs] (TMA staging)
    const uint64_t* rec_off;   // uint4 offset of each record
    // row-per-lane fp32 layout (wbx_sell::rslice / rpk)
    const uint2* rslice;
    const uint4* rpk;
    uint64_t rpk_u4;
    uint32_t rows, xslices, slices;
};

constexpr uint32_t kNoRow = 0xffffffffu;
constexpr uint32_t kRowMask = (1u << 27) - 1;

// Segment partial of this lane, accumulated in ACC with gathers from X.
template <typename ACC, typename X>
__device__ __forceinline__ ACC seg_partial(const SellView& M, uint32_t s, int lane, const X* __restrict__ x) {
    const uint4* p = M.pk + M.slice_ptr[s] + lane;
    const uint32_t np = M.slice_np[s] & 0xffu;
    const uint64_t pol = l2_keep_policy();
    uint4 e[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) e[j] = j < static_cast<int>(np) ? ld_stream(p + j * kWarp, pol) : make_uint4(0, 0, 0, 0);
    X g[16];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (j < static_cast<int>(np)) {
            g[2 * j] = x[e[j].y];
            g[2 * j + 1] = x[e[j].w];
        } else {
            g[2 * j] = X(0);
            g[2 * j + 1] = X(0);
        }
    }
    ACC acc = ACC(0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (j < static_cast<int>(np)) {
            acc = fma(static_cast<ACC>(__uint_as_float(e[j].x)), static_cast<ACC>(g[2 * j]), acc);
            acc = fma(static_cast<ACC>(__uint_as_float(e[j].z)), static_cast<ACC>(g[2 * j + 1]), acc);
        }
    }
    return acc;
}

// Combine segment partials into the head lane; returns the row index (kNoRow for
// non-head lanes) and leaves the row sum in `acc` of the head lane.
template <typename ACC>
__device__ __forceinline__ uint32_t seg_combine(const SellView& M, uint32_t s, int lane, ACC& acc) {
    const uint32_t info = M.lane_info[static_cast<uint64_t>(s) * kWarp + lane];
    const uint32_t m = M.slice_np[s] >> 8;  // lane stride between a row's segments
    const uint32_t nseg = info == kNoRow ? 1u : (info >> 27);
    const uint32_t maxseg = __reduce_max_sync(0xffffffffu, nseg);
    for (uint32_t j = 1; j < maxseg; ++j) {
        const ACC t = __shfl_down_sync(0xffffffffu, acc, j * m);
        if (j < nseg) acc += t;
    }
    return info == kNoRow ? kNoRow : (info & kRowMask);
}

// fp64 values, fp64 vector, reference arithmetic: s = s + v*x, no contraction,
// exactly the row's own elements.
__device__ __forceinline__ double sell_dot_f64_exact(const SellView& M, uint32_t s, int lane,
                                                     const double* __restrict__ x) {
    const uint64_t base = M.xslice_ptr[s] + lane;
    const uint32_t r = s * kWarp + lane;
    const uint32_t len = r < M.rows ? M.row_len[r] : 0;
    const uint64_t pol = l2_keep_policy();
    double acc = 0.0;
    uint32_t j = 0;
    for (; j + 4 <= len; j += 4) {
        const double v0 = ld_stream(M.v64 + base + (j + 0) * kWarp, pol);
        const double v1 = ld_stream(M.v64 + base + (j + 1) * kWarp, pol);
        const double v2 = ld_stream(M.v64 + base + (j + 2) * kWarp, pol);
        const double v3 = ld_stream(M.v64 + base + (j + 3) * kWarp, pol);
        const uint32_t c0 = ld_stream(M.col + base + (j + 0) * kWarp, pol);
        const uint32_t c1 = ld_stream(M.col + base + (j + 1) * kWarp, pol);
        const uint32_t c2 = ld_stream(M.col + base + (j + 2) * kWarp, pol);
        const uint32_t c3 = ld_stream(M.col + base + (j + 3) * kWarp, pol);
        const double g0 = x[c0], g1 = x[c1], g2 = x[c2], g3 = x[c3];
        acc = __dadd_rn(acc, __dmul_rn(v0, g0));
        acc = __dadd_rn(acc, __dmul_rn(v1, g1));
        acc = __dadd_rn(acc, __dmul_rn(v2, g2));
        acc = __dadd_rn(acc, __dmul_rn(v3, g3));
    }
    for (; j < len; ++j) {
        const double v = ld_stream(M.v64 + base + j * kWarp, pol);
        const uint32_t c = ld_stream(M.col + base + j * kWarp, pol);
        acc = __dadd_rn(acc, __dmul_rn(v, x[c]));
    }
    return acc;
}

}  // namespace wbx
