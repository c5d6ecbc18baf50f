// SELL-32 row dot products: one warp per slice, one lane per row.
//
// The lane's row is summed SEQUENTIALLY in element order — the reference's in-row
// order (theta.cpp:306-308) — so the exact fp64 variant reproduces the reference's
// spmv bit for bit; the fp32 variants use FMA and differ only by rounding.
#pragma once

#include "device_util.cuh"

namespace wbx {

struct SellView {
    const uint64_t* slice_ptr;  // pair offset per slice
    const uint32_t* slice_len;  // padded (even) row length of the slice
    const uint4* pk;            // fp32 {v0,c0,v1,c1}
    const double* v64;          // fp64 values, element-major
    const uint32_t* col;        // columns, element-major
    const uint32_t* row_len;    // true row length (fp64 exact path)
    uint32_t rows, slices;
};

// fp32 values, fp32 vector, fp32 FMA accumulation.
__device__ __forceinline__ float sell_dot_f32(const SellView& M, uint32_t s, int lane,
                                              const float* __restrict__ x) {
    const uint4* p = M.pk + M.slice_ptr[s] + lane;
    const uint32_t np = M.slice_len[s] >> 1;
    float acc = 0.f;
    uint32_t j = 0;
    for (; j + 4 <= np; j += 4) {
        const uint4 e0 = ld_stream(p + (j + 0) * kWarp);
        const uint4 e1 = ld_stream(p + (j + 1) * kWarp);
        const uint4 e2 = ld_stream(p + (j + 2) * kWarp);
        const uint4 e3 = ld_stream(p + (j + 3) * kWarp);
        const float g0 = x[e0.y], g1 = x[e0.w], g2 = x[e1.y], g3 = x[e1.w];
        const float g4 = x[e2.y], g5 = x[e2.w], g6 = x[e3.y], g7 = x[e3.w];
        acc = fmaf(__uint_as_float(e0.x), g0, acc);
        acc = fmaf(__uint_as_float(e0.z), g1, acc);
        acc = fmaf(__uint_as_float(e1.x), g2, acc);
        acc = fmaf(__uint_as_float(e1.z), g3, acc);
        acc = fmaf(__uint_as_float(e2.x), g4, acc);
        acc = fmaf(__uint_as_float(e2.z), g5, acc);
        acc = fmaf(__uint_as_float(e3.x), g6, acc);
        acc = fmaf(__uint_as_float(e3.z), g7, acc);
    }
    for (; j < np; ++j) {
        const uint4 e = ld_stream(p + j * kWarp);
        acc = fmaf(__uint_as_float(e.x), x[e.y], acc);
        acc = fmaf(__uint_as_float(e.z), x[e.w], acc);
    }
    return acc;
}

// fp32 values, fp64 vector and accumulation (power iteration in the fp32 hot path).
__device__ __forceinline__ double sell_dot_f32v_f64(const SellView& M, uint32_t s, int lane,
                                                    const double* __restrict__ x) {
    const uint4* p = M.pk + M.slice_ptr[s] + lane;
    const uint32_t np = M.slice_len[s] >> 1;
    double acc = 0.0;
    uint32_t j = 0;
    for (; j + 2 <= np; j += 2) {
        const uint4 e0 = ld_stream(p + (j + 0) * kWarp);
        const uint4 e1 = ld_stream(p + (j + 1) * kWarp);
        const double g0 = x[e0.y], g1 = x[e0.w], g2 = x[e1.y], g3 = x[e1.w];
        acc = fma(static_cast<double>(__uint_as_float(e0.x)), g0, acc);
        acc = fma(static_cast<double>(__uint_as_float(e0.z)), g1, acc);
        acc = fma(static_cast<double>(__uint_as_float(e1.x)), g2, acc);
        acc = fma(static_cast<double>(__uint_as_float(e1.z)), g3, acc);
    }
    for (; j < np; ++j) {
        const uint4 e = ld_stream(p + j * kWarp);
        acc = fma(static_cast<double>(__uint_as_float(e.x)), x[e.y], acc);
        acc = fma(static_cast<double>(__uint_as_float(e.z)), x[e.w], acc);
    }
    return acc;
}

// fp64 values, fp64 vector, reference arithmetic: s = s + v*x, no contraction,
// exactly the row's own elements (no padding terms).
__device__ __forceinline__ double sell_dot_f64_exact(const SellView& M, uint32_t s, int lane,
                                                     const double* __restrict__ x) {
    const uint64_t base = 2 * M.slice_ptr[s] + lane;
    const uint32_t r = s * kWarp + lane;
    const uint32_t len = r < M.rows ? M.row_len[r] : 0;
    double acc = 0.0;
    uint32_t j = 0;
    for (; j + 4 <= len; j += 4) {
        const double v0 = ld_stream(M.v64 + base + (j + 0) * kWarp);
        const double v1 = ld_stream(M.v64 + base + (j + 1) * kWarp);
        const double v2 = ld_stream(M.v64 + base + (j + 2) * kWarp);
        const double v3 = ld_stream(M.v64 + base + (j + 3) * kWarp);
        const uint32_t c0 = ld_stream(M.col + base + (j + 0) * kWarp);
        const uint32_t c1 = ld_stream(M.col + base + (j + 1) * kWarp);
        const uint32_t c2 = ld_stream(M.col + base + (j + 2) * kWarp);
        const uint32_t c3 = ld_stream(M.col + base + (j + 3) * kWarp);
        const double g0 = x[c0], g1 = x[c1], g2 = x[c2], g3 = x[c3];
        acc = __dadd_rn(acc, __dmul_rn(v0, g0));
        acc = __dadd_rn(acc, __dmul_rn(v1, g1));
        acc = __dadd_rn(acc, __dmul_rn(v2, g2));
        acc = __dadd_rn(acc, __dmul_rn(v3, g3));
    }
    for (; j < len; ++j) {
        const double v = ld_stream(M.v64 + base + j * kWarp);
        const uint32_t c = ld_stream(M.col + base + j * kWarp);
        acc = __dadd_rn(acc, __dmul_rn(v, x[c]));
    }
    return acc;
}

}  // namespace wbx
