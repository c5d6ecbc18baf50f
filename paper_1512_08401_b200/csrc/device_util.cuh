// Small device helpers shared by the SpMV and solver kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace wbx {

constexpr int kWarp = 32;

// Loads of the read-only operator streams: bypass L1 allocation (each element is read
// once per SM per iteration, the L1 is kept for the gathered vector entries, which ARE
// reused across lanes and rows) and mark the lines EVICT_LAST in L2 so the operator
// (tens of MB) stays resident in the 126 MB L2 across solver iterations. A plain
// `.nc.L1::no_allocate` load is treated as evict-first by L2 and re-streams from HBM
// every iteration (ncu: 72 % L2 miss on those sectors).
__device__ __forceinline__ uint64_t l2_keep_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint4 ld_stream(const uint4* p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint2 ld_stream(const uint2* p, uint64_t pol) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_stream(const uint16_t* p, uint64_t pol) {
    unsigned short r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Sense-free generation barrier across all co-resident blocks of a cooperative launch.
// bar[0] = arrival count (returns to 0 after every barrier), bar[1] = generation.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire(bar + 1);
        __threadfence();
        const unsigned prev = atomicAdd(bar, 1u);
        if (prev == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (ld_acquire(bar + 1) == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum (fixed tree), result valid in every thread.
template <int kThreads>
__device__ __forceinline__ double block_sum(double v, double* smem) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < kThreads / 32 ? smem[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) smem[0] = t;
    }
    __syncthreads();
    const double r = smem[0];
    __syncthreads();
    return r;
}

// Deterministic sum of `count` per-block partials (same result in every block).
__device__ __forceinline__ double reduce_partials(const double* part, unsigned count,
                                                  double* smem) {
    double v = 0.0;
    if (threadIdx.x < 32) {
        for (unsigned i = threadIdx.x; i < count; i += 32) v += part[i];
        v = warp_sum(v);
        if (threadIdx.x == 0) smem[0] = v;
    }
    __syncthreads();
    const double r = smem[0];
    __syncthreads();
    return r;
}

}  // namespace wbx
