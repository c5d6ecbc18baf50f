// Per-warp TMA (cp.async.bulk) prefetch of the operator streams into shared memory.
//
// In the persistent solver every warp owns a fixed list of SELL slices of Theta
// ("A", phase A) and of Theta^T ("T", phase T). Its operator data for one iteration is
// therefore a fixed, periodic sequence of contiguous byte ranges:
//     A_0 .. A_{nA-1}, T_0 .. T_{nT-1}, A_0, ...
// independent of the iteration's values. Lane 0 keeps the next kSlots entries of that
// sequence in flight as 1-D bulk copies (the TMA engine, no registers held), each
// completing on its own mbarrier; the warp consumes entries in order from shared memory.
// The copies for the NEXT phase are issued while the current phase computes and while the
// warp waits at the grid barrier, so the operator loads leave the critical path: a slice
// costs one round trip (its vector gathers) instead of two.
#pragma once

#include "device_util.cuh"

namespace wbx {

constexpr int kSlots = 3;                       // in-flight slices per warp
constexpr unsigned kSlotBytes = 8u * 32u * 16u; // max slice: 8 pairs x 32 lanes x 16 B

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// 1-D bulk copy global -> shared (TMA engine), completion as transaction bytes on `bar`,
// L2 eviction hint `pol` (the operator is re-read every iteration: evict_last).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Per-warp slot ring in shared memory.
struct WarpRing {
    uint4* slot;     // kSlots * (kSlotBytes / 16) uint4
    uint64_t* bar;   // kSlots mbarriers
};

}  // namespace wbx
