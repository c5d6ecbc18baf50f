// Preconditioned FISTA / ISTA on the device: persistent cooperative kernels.
//
// Replaces run_pgd (`proj/src/solver.cpp:103-157`), estimate_step (:69-99) and
// prox_weighted_l1_P (:57-67). Per iteration the reference does 3 CSR SpMVs and ~6
// serial O(n) passes with fresh allocations; here a solve is TWO resident kernels:
//
//   tau_kernel   (estimate_step): per power iteration
//       phase A  t = Theta u / |w_prev|         (rows R)      -- grid barrier --
//       phase T  w = P^-1/2 Theta^T t; <v,w>, <w,w>  (rows C of Theta^T) -- barrier+reduction --
//   fista_kernel (run_pgd loop): per iteration
//       phase A  res[r] = (Theta y)[r] - x0[r]                           -- grid barrier --
//       phase T  g = (Theta^T res)[c]; z0 = y - tau g / p; x' = prox(z0);
//                y = x' + beta_k (x' - x_prev)                             -- grid barrier --
//     i.e. gradient + residual + preconditioner + weighted soft threshold + momentum
//     fused into the Theta^T SpMV epilogue.
//
// Vectors live in COMPACTED coordinates (R = nonempty rows, C = nonempty columns);
// every other coordinate has gradient exactly 0 (empty column of Theta), so its
// trajectory is the 1-D recurrence x' = prox(y), y = x' + beta (x' - x_prev): those are
// iterated to completion in registers in one pass (loop interchange; per-coordinate
// arithmetic identical to the reference's).
//
// Each warp owns a fixed set of SELL slices for the whole solve; their metadata is
// loaded once into registers, so an iteration's dependency chain per slice is the
// operator load + the gather. The grid barrier is a flag barrier (one arrival word per
// block, no atomics) whose master block also performs the deterministic grid reduction.
//
// Precision: WBX_FP32 is the hot path (fp32 values/vectors, FMA); WBX_FP64 reproduces
// the reference arithmetic exactly (sequential in-row sums, no contraction, the
// reference's expression order) and, given the same tau, its iterates BITWISE.
// tau uses fp64 vectors and accumulation in both modes (fp32 or fp64 operator values)
// with the reference's CounterRng(0x5eed) start, 200-iteration cap and 1e-6 rule.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <list>

#include "internal.hpp"
#include "wbx_diag.h"
#include "sell.cuh"
#include "stream.cuh"
#include "win.cuh"
#include "lanczos.cuh"
#include "stencil_engine.cuh"
#include "rng.cuh"

extern "C" void wbx_set_last_error(const char* msg);

namespace wbx {

namespace {

constexpr int kBlock = 256;
constexpr int kWarpsPerBlock = kBlock / 32;
constexpr int kMaxK = 8;        // slices per warp kept in registers
constexpr int kRedSlots = 4;    // values per grid reduction
#ifndef WBX_FISTA_MINB
#define WBX_FISTA_MINB 2
#endif
#ifndef WBX_TAU_MINB
#define WBX_TAU_MINB 2
#endif

// output scalars (SolveArgs::out)
enum : int {
    OUT_TAU = 0,
    OUT_TAU_ITERS = 1,
    OUT_ITERS_USED = 2,
    OUT_INITIAL_ENERGY = 3,
    OUT_STATUS = 4,  // 0 ok, 8 nonfinite energy
    OUT_LAMBDA_MAX = 5,
    OUT_TAU_STEPS = 6,  // operator products (pairs) spent on tau: power iterations or Lanczos steps
    OUT_COUNT = 8
};

// Grid barrier state (device memory, zeroed once per solver).
struct Sync {
    unsigned* gen;     // released epoch
    unsigned* arrive;  // [grid] arrived epoch per block
    double* part;      // [kRedSlots][grid] block partials
    double* red;       // [kRedSlots] grid totals of the last reduction
    unsigned long long* trace;  // optional [trace_cap][grid][2] globaltimer stamps
    unsigned trace_cap;
    int mode;  // 0: master block releases, 1: every block polls all arrivals, 2: counter (default)
    int groups;  // counter barrier: arrival counters (one 128-B line each; block b uses b % groups)
};

struct SolveArgs {
    SellView A, T;
    const uint32_t* R_glob;
    const uint32_t* C_glob;
    const uint32_t* isC;
    const uint32_t* isR;
    uint32_t nR, nC;
    uint64_t n;
    const double* x0_full;
    const double* w_full;
    const double* p_full;
    double* x_full;
    const double* pC;
    const double* wC;
    const double* ispC;
    const double* beta64;  // beta_k, k = 1..max_iters (index k-1)
    const float* beta32;
    double lambda, tau_given, step_safety, ref_energy, rel_tol;
    int tau_from_device, max_iters, track, stop_on_ref, decoupled_inline, nslots;
    // window engine (win.cuh): per-CTA layouts of Theta (A) and Theta^T (T)
    WinView wA, wT;
    int lz_first, lz_every, lz_gap;  // Lanczos tau: first check, check period, compared m - gap
    double lz_tol;                   // Lanczos tau: two checks agree when lambda is within lz_tol
    int win_lists_global;            // window index lists read from global memory (win_smem_head)
    // stencil engine (stencil_engine.cuh): the plan and its fp32 source vectors
    StencilView st;
    int st_fill;  // window fill: 0 bulk copies (TMA), 1 cp.async 16 B per warp row (WBX_ST_FILL)
    float* yF;
    float* resF;
    // T-typed state
    void* yC;
    void* xpC;
    void* res;
    void* x0R;
    void* tpC;
    void* thrC;
    // power iteration (fp64)
    double* wv;
    double* uC;
    double* t64;
    const double* dec_reg;   // [max_iters] decoupled sum w|x_k| (tracking)
    const double* dec_supp;  // [max_iters] decoupled support count (tracking)
    double* out;
    double* energies;
    unsigned long long* supports;
    Sync sync;
};

__device__ __forceinline__ bool bit_set(const uint32_t* mask, uint64_t i) {
    return (mask[i >> 5] >> (i & 31)) & 1u;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}


// Master warp: poll all arrival words, every lane its strided subset with independent
// loads per round (one memory round trip per round, not one per block), then acquire.
__device__ __forceinline__ void wait_arrivals(const Sync& s, unsigned epoch, unsigned G) {
    constexpr int kMaxPoll = 40;  // grids up to 1280 blocks
    bool ok;
    do {
        unsigned v[kMaxPoll];
#pragma unroll
        for (int j = 0; j < kMaxPoll; ++j) {
            const unsigned i = threadIdx.x + 32u * j;
            v[j] = i < G ? ld_relaxed(s.arrive + i) : epoch;
        }
        ok = true;
#pragma unroll
        for (int j = 0; j < kMaxPoll; ++j) ok &= static_cast<int>(v[j] - epoch) >= 0;
    } while (!__all_sync(0xffffffffu, ok));
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// ---------------------------------------------------------------- grid barrier + reduction
// Arrival: each block publishes its partials and then its epoch in its own word (no
// atomics). Block 0's first warp waits for every word, reduces the partials in a fixed
// order, publishes the totals and releases the epoch; the other blocks spin on it.
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Barrier epoch of this block; `start` is the released epoch seen at kernel entry.
struct Epoch {
    unsigned cur, start;
};

// Back-off between barrier polls (ns; 0 = spin)
#ifndef WBX_POLL_NS
#define WBX_POLL_NS 0
#endif

// Counter barrier (mode 2): one arrival counter, zeroed by the host before each cooperative
// launch; barrier k of the launch completes when the counter reaches k * G. Arrival is a
// fire-and-forget reduction, and every block polls the one word directly (no master hop).
constexpr unsigned kCounterWord = 32;  // Sync::gen[kCounterWord + 32 g]: counter g, its own 128-B line
constexpr int kMaxCounterGroups = 16;

// Warp 0 of every block (all 32 lanes call it): arrive on the block's group counter, then wait
// until every group counter has reached its share of k * G. With groups > 1 the arrivals spread
// over several L2 lines (the same-address reductions of one counter serialise at its L2 slice);
// lane g polls counter g, one round trip per poll round.
__device__ __forceinline__ void counter_arrive_wait(const Sync& s, const Epoch& e) {
    unsigned* cnt = s.gen + kCounterWord;
    const int ng = s.groups;
    const unsigned G = gridDim.x, k = e.cur - e.start;
    const unsigned lane = threadIdx.x & 31;
    if (lane == 0)
        asm volatile("fence.acq_rel.gpu;\nred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + 32u * (blockIdx.x % ng))
                     : "memory");
    const unsigned members = G / ng + (lane < G % ng ? 1u : 0u);
    const unsigned target = k * members;
    bool ok;
    // acquiring polls: measured faster than relaxed polls + one acquire fence (the fence
    // costs more than the per-poll L1 invalidations)
    do {
        ok = true;
        if (lane < static_cast<unsigned>(ng)) ok = static_cast<int>(ld_acquire(cnt + 32u * lane) - target) >= 0;
        if (WBX_POLL_NS && !__all_sync(0xffffffffu, ok)) __nanosleep(WBX_POLL_NS);
    } while (!__all_sync(0xffffffffu, ok));
}

// Optional phase trace (WBX_TRACE_FILE): per barrier and block, the time the block
// arrived and the time it saw the release.
__device__ __forceinline__ void trace_point(const Sync& s, const Epoch& e, int which) {
    if (s.trace != nullptr && threadIdx.x == 0) {
        const unsigned idx = e.cur - e.start - 1;
        if (idx < s.trace_cap) s.trace[(static_cast<uint64_t>(idx) * gridDim.x + blockIdx.x) * 2 + which] = globaltimer();
    }
}

// All-poll barrier: a block arrives by publishing (partials, then) its epoch in its own
// word; the first warp of EVERY block polls all arrival words (one batched round trip
// per poll round) — no master hop, no atomics. Reductions: every block sums the
// published block partials itself in the same fixed order, so all blocks obtain
// bit-identical totals. Partials are double-buffered by epoch parity (a block cannot
// run two barriers ahead of any other block).
template <int NV, int BS = kBlock>
__device__ __forceinline__ void grid_sync_reduce(const Sync& s, Epoch& epoch, double (&v)[NV],
                                                 double* smem) {
    const unsigned G = gridDim.x;
    ++epoch.cur;
    double* part = s.part + static_cast<uint64_t>(epoch.cur & 1u) * kRedSlots * G;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const double b = block_sum<BS>(v[k], smem);
        if (threadIdx.x == 0) part[k * G + blockIdx.x] = b;
    }
    trace_point(s, epoch, 0);
    if (s.mode == 2) {  // counter barrier, then every block reduces the partials itself
        __syncthreads();
        if (threadIdx.x < 32) counter_arrive_wait(s, epoch);
        __syncthreads();
        if (threadIdx.x < 32) {
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                double t = 0.0;
                for (unsigned i = threadIdx.x; i < G; i += 32) t += part[k * G + i];
                t = warp_sum(t);
                if (threadIdx.x == 0) smem[k] = t;
            }
        }
        trace_point(s, epoch, 1);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] = smem[k];
        __syncthreads();
        return;
    }
    if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        st_release(s.arrive + blockIdx.x, epoch.cur);
    }
    if (s.mode == 1) {  // all-poll: every block reduces
        if (threadIdx.x < 32) {
            wait_arrivals(s, epoch.cur, G);
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                double t = 0.0;
                for (unsigned i = threadIdx.x; i < G; i += 32) t += part[k * G + i];
                t = warp_sum(t);
                if (threadIdx.x == 0) smem[k] = t;
            }
        }
    } else {  // master: block 0 reduces, publishes, releases
        if (blockIdx.x == 0 && threadIdx.x < 32) {
            wait_arrivals(s, epoch.cur, G);
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                double t = 0.0;
                for (unsigned i = threadIdx.x; i < G; i += 32) t += part[k * G + i];
                t = warp_sum(t);
                if (threadIdx.x == 0) s.red[k] = t;
            }
            __syncwarp();
            if (threadIdx.x == 0) st_release(s.gen, epoch.cur);
        }
        if (threadIdx.x == 0) {
            while (static_cast<int>(ld_acquire(s.gen) - epoch.cur) < 0) {
            }
#pragma unroll
            for (int k = 0; k < NV; ++k) smem[k] = s.red[k];
        }
    }
    trace_point(s, epoch, 1);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = smem[k];
    __syncthreads();
}

__device__ __forceinline__ void grid_sync(const Sync& s, Epoch& epoch, double* smem) {
    const unsigned G = gridDim.x;
    ++epoch.cur;
    __syncthreads();
    trace_point(s, epoch, 0);
    if (s.mode == 2) {
        if (threadIdx.x < 32) counter_arrive_wait(s, epoch);
        trace_point(s, epoch, 1);
        __syncthreads();
        return;
    }
    if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        st_release(s.arrive + blockIdx.x, epoch.cur);
    }
    if (s.mode == 1) {
        if (threadIdx.x < 32) wait_arrivals(s, epoch.cur, G);
    } else {
        if (blockIdx.x == 0 && threadIdx.x < 32) {
            wait_arrivals(s, epoch.cur, G);
            if (threadIdx.x == 0) st_release(s.gen, epoch.cur);
        }
        if (threadIdx.x == 0)
            while (static_cast<int>(ld_acquire(s.gen) - epoch.cur) < 0) {
            }
    }
    trace_point(s, epoch, 1);
    (void)smem;
    __syncthreads();
}

// ---------------------------------------------------------------- per-warp slice plan
// The slices a warp owns (s = gwarp + k * nwarps) with their metadata in registers:
// lane k holds slice k's pair offset and pair count, every lane its own lane_info word
// for each slice. Falls back to per-slice metadata loads beyond kMaxK slices.
struct Plan {
    uint32_t nk;
    uint32_t np;
    uint64_t ptr;
    uint32_t info[kMaxK];
    bool fallback;
};

__device__ __forceinline__ Plan make_plan(const SellView& M, uint32_t gwarp, uint32_t nwarps, int lane) {
    Plan p;
    p.nk = M.slices > gwarp ? (M.slices - gwarp + nwarps - 1) / nwarps : 0;
    p.fallback = p.nk > kMaxK;
    p.np = 0;
    p.ptr = 0;
    if (!p.fallback && static_cast<uint32_t>(lane) < p.nk) {
        const uint32_t s = gwarp + lane * nwarps;
        p.ptr = M.slice_ptr[s];
        p.np = M.slice_np[s];
    }
#pragma unroll
    for (int k = 0; k < kMaxK; ++k)
        p.info[k] = (!p.fallback && static_cast<uint32_t>(k) < p.nk)
                        ? M.lane_info[static_cast<uint64_t>(gwarp + k * nwarps) * kWarp + lane]
                        : kNoRow;
    return p;
}

// Segment partial with explicit slice base / pair count (see seg_partial in sell.cuh).
template <typename ACC, typename X>
__device__ __forceinline__ ACC seg_partial_at(const uint4* __restrict__ p, uint32_t np,
                                              const X* __restrict__ x, uint64_t pol) {
    uint4 e[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) e[j] = j < static_cast<int>(np) ? ld_stream(p + j * kWarp, pol) : make_uint4(0, 0, 0, 0);
    X g[16];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        g[2 * j] = j < static_cast<int>(np) ? x[e[j].y] : X(0);
        g[2 * j + 1] = j < static_cast<int>(np) ? x[e[j].w] : X(0);
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

// meta = slice_np word: pairs per lane (bits 0-7) | lane stride m of a row's segments
template <typename ACC>
__device__ __forceinline__ uint32_t combine_info(uint32_t info, uint32_t meta, ACC& acc) {
    const uint32_t m = meta >> 8;
    const uint32_t nseg = info == kNoRow ? 1u : (info >> 27);
    const uint32_t maxseg = __reduce_max_sync(0xffffffffu, nseg);
    for (uint32_t j = 1; j < maxseg; ++j) {
        const ACC t = __shfl_down_sync(0xffffffffu, acc, j * m);
        if (j < nseg) acc += t;
    }
    return info == kNoRow ? kNoRow : (info & kRowMask);
}

// Apply `epi(row, value)` to every row of the warp's slices: value = sum_j M[row,j] x[j]
// accumulated in ACC over the segmented fp32 layout.
template <typename ACC, typename X, typename Epi>
__device__ __forceinline__ void for_rows_seg(const SellView& M, const Plan& plan, uint32_t gwarp, uint32_t nwarps,
                                             int lane, const X* __restrict__ x, Epi epi) {
    const uint64_t pol = l2_keep_policy();
    if (!plan.fallback) {
#pragma unroll
        for (int k = 0; k < kMaxK; ++k) {
            if (static_cast<uint32_t>(k) >= plan.nk) break;
            const uint64_t ptr = __shfl_sync(0xffffffffu, plan.ptr, k);
            const uint32_t meta = __shfl_sync(0xffffffffu, plan.np, k);
            ACC acc = seg_partial_at<ACC, X>(M.pk + ptr + lane, meta & 0xffu, x, pol);
            const uint32_t row = combine_info(plan.info[k], meta, acc);
            if (row != kNoRow) epi(row, acc);
        }
    } else {
        for (uint32_t s = gwarp; s < M.slices; s += nwarps) {
            const uint32_t meta = M.slice_np[s];
            ACC acc = seg_partial_at<ACC, X>(M.pk + M.slice_ptr[s] + lane, meta & 0xffu, x, pol);
            const uint32_t row = combine_info(M.lane_info[static_cast<uint64_t>(s) * kWarp + lane], meta, acc);
            if (row != kNoRow) epi(row, acc);
        }
    }
}

// Same over the exact fp64 layout (one lane per row, reference order).
template <typename Epi>
__device__ __forceinline__ void for_rows_exact(const SellView& M, uint32_t gwarp, uint32_t nwarps, int lane,
                                               const double* __restrict__ x, Epi epi) {
    for (uint32_t s = gwarp; s < M.xslices; s += nwarps) {
        const double v = sell_dot_f64_exact(M, s, lane, x);
        const uint32_t r = s * kWarp + lane;
        if (r < M.rows) epi(r, v);
    }
}

// ---------------------------------------------------------------- precision traits
template <typename T>
struct Prec;

template <>
struct Prec<float> {
    __device__ static float sub(float a, float b) { return a - b; }
    // z0 = y - (tau/p) g   (tp = tau/p precomputed in fp64, rounded once)
    __device__ static float z0(float y, float g, float tp, double, double) { return fmaf(-tp, g, y); }
    __device__ static float prox(float z0, float thr) {
        const float a = fabsf(z0) - thr;
        return a > 0.f ? (z0 > 0.f ? a : -a) : 0.f;
    }
    __device__ static float momentum(float xn, float xp, float beta) { return fmaf(beta, xn - xp, xn); }
    __device__ static float beta(const SolveArgs& a, int k) { return a.beta32[k - 1]; }
};

template <>
struct Prec<double> {
    __device__ static double sub(double a, double b) { return __dsub_rn(a, b); }
    // solver.cpp:126: y - tau * grad / p  ==  y - ((tau*grad)/p)
    __device__ static double z0(double y, double g, double, double tau, double p) {
        return __dsub_rn(y, __ddiv_rn(__dmul_rn(tau, g), p));
    }
    // solver.cpp:62-64
    __device__ static double prox(double z0, double thr) {
        const double a = __dsub_rn(fabs(z0), thr);
        return a > 0.0 ? (z0 > 0.0 ? a : -a) : 0.0;
    }
    // solver.cpp:145: x_new + beta * (x_new - x_prev)
    __device__ static double momentum(double xn, double xp, double beta) {
        return __dadd_rn(xn, __dmul_rn(beta, __dsub_rn(xn, xp)));
    }
    __device__ static double beta(const SolveArgs& a, int k) { return a.beta64[k - 1]; }
};

// thr = tau * lambda * w / p, evaluated left to right as the reference (solver.cpp:61)
__device__ __forceinline__ double thr_exact(double tau, double lambda, double w, double p) {
    return __ddiv_rn(__dmul_rn(__dmul_rn(tau, lambda), w), p);
}

// Row loop dispatch: T = float -> segmented fp32 values (ACC/X as given);
// T = double -> exact fp64 layout.
template <typename T, typename ACC, typename X, typename Epi>
__device__ __forceinline__ void for_rows(const SellView& M, const Plan& plan, uint32_t gwarp, uint32_t nwarps,
                                         int lane, const X* x, Epi epi) {
    if constexpr (sizeof(T) == 4) {
        for_rows_seg<ACC, X>(M, plan, gwarp, nwarps, lane, x, epi);
    } else {
        for_rows_exact(M, gwarp, nwarps, lane, reinterpret_cast<const double*>(x), epi);
    }
}

// ---------------------------------------------------------------- decoupled coordinates
// Coordinates with an empty Theta column: g == 0 exactly, so z0 == y and the iterate
// is prox + momentum only. Runs K iterations per coordinate in registers and stops as
// soon as x' == x_prev == 0 (then y == 0 forever: a fixed point).
// mode 0: write x_K into x_full.  mode 1: per-iteration warp sums of w|x_k| and
// [x_k != 0] into w*[(k-1) * nwarps + gwarp] (deterministic, no atomics). mode 2: both
// (the iteration count is known in advance: no ref_energy rule).
template <typename T>
__device__ void decoupled_pass(const SolveArgs& a, double tau, int K, int mode, uint64_t gthread,
                               uint64_t nthreads, double* wreg, double* wsup, uint64_t nwarps) {
    const int lane = threadIdx.x & 31;
    const uint64_t gwarp = gthread >> 5;
    const uint64_t trips = (a.n + nthreads - 1) / nthreads;  // warp-uniform
    for (uint64_t t = 0; t < trips; ++t) {
        const uint64_t i = t * nthreads + gthread;
        const bool active = i < a.n && !bit_set(a.isC, i);
        T x = T(0), xp = T(0), y = T(0);
        T thr = T(0);
        double w = 0.0;
        if (active) {
            const double x0 = a.x0_full[i];
            w = a.w_full[i];
            thr = static_cast<T>(thr_exact(tau, a.lambda, w, a.p_full[i]));
            x = xp = y = static_cast<T>(x0);
        }
        if (mode == 0) {
            if (active) {
                for (int k = 1; k <= K; ++k) {
                    const T xn = Prec<T>::prox(y, thr);
                    const bool fixed = xn == T(0) && xp == T(0);
                    y = Prec<T>::momentum(xn, xp, Prec<T>::beta(a, k));
                    xp = xn;
                    x = xn;
                    if (fixed) break;
                }
                a.x_full[i] = static_cast<double>(x);
            }
        } else {
            bool live = active;
            for (int k = 1; k <= K; ++k) {
                double reg = 0.0, sup = 0.0;
                if (live) {
                    const T xn = Prec<T>::prox(y, thr);
                    const bool fixed = xn == T(0) && xp == T(0);
                    y = Prec<T>::momentum(xn, xp, Prec<T>::beta(a, k));
                    xp = xn;
                    x = xn;
                    reg = w * fabs(static_cast<double>(xn));
                    sup = xn != T(0) ? 1.0 : 0.0;
                    if (fixed) live = false;
                }
                reg = warp_sum(reg);
                sup = warp_sum(sup);
                if (lane == 0) {
                    wreg[static_cast<uint64_t>(k - 1) * nwarps + gwarp] += reg;
                    wsup[static_cast<uint64_t>(k - 1) * nwarps + gwarp] += sup;
                }
                if (!__any_sync(0xffffffffu, live)) break;
            }
            if (mode == 2 && active) a.x_full[i] = static_cast<double>(x);
        }
    }
}

// Debug build (make check): bounds assertions in the window engine; a violation traps the
// kernel (the call then fails with a CUDA error) instead of reading or writing out of range.
#ifndef WBX_CHECKS
#define WBX_CHECKS 0
#endif
#define WBX_ASSERT(cond)                       \
    do {                                       \
        if (WBX_CHECKS && !(cond)) __trap();   \
    } while (0)

// Compile-time diagnostics (make prof, WBX_PROFILE=3): cycle accounting of the window engine
// (wbx_diag_slice_profile, tools/win_profile.py)
#ifndef WBX_PROFILE
#define WBX_PROFILE 0
#endif
#ifndef WBX_TAU_ACC32
#define WBX_TAU_ACC32 1
#endif
// Per-lane register cache of the last dictionary block (single-slice mode)
#ifndef WBX_DICT_CACHE
#define WBX_DICT_CACHE 1
#endif
__device__ unsigned long long g_prof[8];

}  // namespace
}  // namespace wbx

extern "C" int wbx_diag_slice_profile(double* out) {
    unsigned long long h[8];
    if (cudaMemcpyFromSymbol(h, wbx::g_prof, sizeof h) != cudaSuccess) return WBX_CUDA_ERROR;
    for (int i = 0; i < 8; ++i) out[i] = static_cast<double>(h[i]);  // raw cycle totals (WinProf)
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(wbx::g_prof, z, sizeof z);
    return WBX_OK;
}

namespace wbx {
namespace {

// ---------------------------------------------------------------- TMA-staged operator stream
// Per-warp ring of kSlots slice records in shared memory filled by 1-D bulk copies
// (stream.cuh). Entry e of the warp's periodic sequence (period P = nA + nT [+ nA when
// the energy pass is on]) is slice k of Theta (A) or Theta^T (T).
constexpr unsigned kRecU4 = (kSlotBytes + 128u) / 16u;  // slot stride in uint4 (max record)
constexpr int kMaxSlots = 8;
// per-warp shared memory: [mbarriers x8][meta x8][pad to 128][ns x record slot]
__host__ __device__ constexpr unsigned warp_smem_bytes(int ns) { return 128u + static_cast<unsigned>(ns) * kRecU4 * 16u; }

struct Streamer {
    uint4* slots;
    uint64_t* bars;
    uint32_t* meta;
    uint32_t ns;  // slots in flight (<= kMaxSlots)
    uint32_t nA, nT, P;
    uint64_t issued, consumed, limit;
    uint64_t pol;
    // lane j holds the metadata of period entry j (P <= 32), so issuing never waits on
    // a global load
    uint32_t reg_meta;
    uint64_t reg_off;
    // P > 32: lane j holds the metadata of entry 32w + j of the current issue window w and
    // of the next one (one coalesced load per 32 issues, a window ahead of its use)
    uint32_t cur_meta, nx_meta;
    uint64_t cur_off, nx_off;
};

__device__ __forceinline__ uint32_t count_slices(const SellView& M, uint32_t gwarp, uint32_t nwarps) {
    return M.slices > gwarp ? (M.slices - gwarp + nwarps - 1) / nwarps : 0;
}

// entry r of the period -> (operator, slice)
__device__ __forceinline__ uint32_t entry_slice(const Streamer& st, uint32_t r, uint32_t gwarp, uint32_t nwarps,
                                                bool& isT) {
    isT = r >= st.nA && r < st.nA + st.nT;
    const uint32_t k = r < st.nA ? r : (isT ? r - st.nA : r - st.nA - st.nT);
    return gwarp + k * nwarps;
}

__device__ __forceinline__ void st_load_window(Streamer& st, const SellView& A, const SellView& T, uint32_t gwarp,
                                               uint32_t nwarps, int lane, uint64_t first) {
    const uint64_t e = first + static_cast<uint64_t>(lane);
    st.nx_meta = 0;
    st.nx_off = 0;
    if (e < st.limit) {
        bool isT;
        const uint32_t s = entry_slice(st, static_cast<uint32_t>(e % st.P), gwarp, nwarps, isT);
        const SellView& M = isT ? T : A;
        st.nx_meta = M.slice_np[s];
        st.nx_off = M.rec_off[s];
    }
}

__device__ __forceinline__ void st_issue(Streamer& st, const SellView& A, const SellView& T, uint32_t gwarp,
                                         uint32_t nwarps, int lane) {
    const uint64_t e = st.issued++;
    const uint32_t r = static_cast<uint32_t>(e % st.P);
    bool isT;
    entry_slice(st, r, gwarp, nwarps, isT);
    const SellView& M = isT ? T : A;
    uint32_t meta;
    uint64_t off;
    if (st.P <= 32) {
        meta = __shfl_sync(0xffffffffu, st.reg_meta, r);
        off = __shfl_sync(0xffffffffu, st.reg_off, r);
    } else {
        if ((e & 31u) == 0 && e > 0) {  // next window: the prefetched one becomes current
            st.cur_meta = st.nx_meta;
            st.cur_off = st.nx_off;
            st_load_window(st, A, T, gwarp, nwarps, lane, e + 32);
        }
        meta = __shfl_sync(0xffffffffu, st.cur_meta, static_cast<int>(e & 31u));
        off = __shfl_sync(0xffffffffu, st.cur_off, static_cast<int>(e & 31u));
    }
    if (lane != 0) return;
    const unsigned bytes = 128u + (meta & 0xffu) * 512u;
    const unsigned slot = static_cast<unsigned>(e % st.ns);
    st.meta[slot] = meta;
    mbar_expect_tx(st.bars + slot, bytes);
    bulk_g2s(st.slots + slot * kRecU4, M.rec + off, bytes, st.bars + slot, st.pol);
}

__device__ __forceinline__ void st_init(Streamer& st, unsigned char* warp_smem, const SellView& A,
                                        const SellView& T, uint32_t gwarp, uint32_t nwarps, int lane,
                                        uint64_t iters, bool energy_pass, int nslots) {
    st.bars = reinterpret_cast<uint64_t*>(warp_smem);
    st.meta = reinterpret_cast<uint32_t*>(warp_smem + 8u * kMaxSlots);
    st.slots = reinterpret_cast<uint4*>(warp_smem + 128u);
    st.ns = static_cast<uint32_t>(nslots);
    st.nA = count_slices(A, gwarp, nwarps);
    st.nT = count_slices(T, gwarp, nwarps);
    st.P = st.nA + st.nT + (energy_pass ? st.nA : 0);
    st.issued = st.consumed = 0;
    st.limit = st.P == 0 ? 0 : iters * st.P;
    st.pol = l2_keep_policy();
    st.reg_meta = 0;
    st.reg_off = 0;
    if (st.P <= 32 && static_cast<uint32_t>(lane) < st.P) {
        bool isT;
        const uint32_t s = entry_slice(st, static_cast<uint32_t>(lane), gwarp, nwarps, isT);
        const SellView& M = isT ? T : A;
        st.reg_meta = M.slice_np[s];
        st.reg_off = M.rec_off[s];
    }
    if (lane == 0)
        for (uint32_t i = 0; i < st.ns; ++i) mbar_init(st.bars + i, 1);
    mbar_fence_init();
    __syncwarp();
    if (st.P > 32) {
        st_load_window(st, A, T, gwarp, nwarps, lane, 0);
        st.cur_meta = st.nx_meta;
        st.cur_off = st.nx_off;
        st_load_window(st, A, T, gwarp, nwarps, lane, 32);
    }
    while (st.issued < st.limit && st.issued < st.ns) st_issue(st, A, T, gwarp, nwarps, lane);
}

// Consume the next `count` entries: value = sum over the row of val * x[col] (ACC
// accumulation), combined over the row's segments. pre(row) issues the epilogue's own
// loads BEFORE the gathers (same round trip); post(row, value, pre) runs on head lanes.
template <typename ACC, typename X, typename Pre, typename Post>
__device__ __forceinline__ void st_phase(Streamer& st, const SellView& A, const SellView& T, uint32_t gwarp,
                                         uint32_t nwarps, int lane, uint32_t count, const X* __restrict__ x,
                                         Pre pre, Post post) {
    for (uint32_t i = 0; i < count; ++i) {
        const uint64_t e = st.consumed;
        const unsigned slot = static_cast<unsigned>(e % st.ns);
        mbar_wait(st.bars + slot, static_cast<unsigned>((e / st.ns) & 1u));
        const uint32_t meta = st.meta[slot];
        const uint32_t np = meta & 0xffu;
        const uint4* rec = st.slots + slot * kRecU4;
        const uint32_t info = reinterpret_cast<const uint32_t*>(rec)[lane];
        const auto pv = pre(info == kNoRow ? kNoRow : (info & kRowMask));
        const uint4* p = rec + 8 + lane;
        uint4 q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = j < static_cast<int>(np) ? p[j * kWarp] : make_uint4(0, 0, 0, 0);
        X g[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            g[2 * j] = j < static_cast<int>(np) ? x[q[j].y] : X(0);
            g[2 * j + 1] = j < static_cast<int>(np) ? x[q[j].w] : X(0);
        }
        ACC acc = ACC(0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j < static_cast<int>(np)) {
                acc = fma(static_cast<ACC>(__uint_as_float(q[j].x)), static_cast<ACC>(g[2 * j]), acc);
                acc = fma(static_cast<ACC>(__uint_as_float(q[j].z)), static_cast<ACC>(g[2 * j + 1]), acc);
            }
        }
        const uint32_t row = combine_info(info, meta, acc);
        __syncwarp();  // every lane is done with the slot before it is refilled
        st.consumed = e + 1;
        if (st.issued < st.limit) st_issue(st, A, T, gwarp, nwarps, lane);
        if (row != kNoRow) post(row, acc, pv);
    }
}

// Wait for copies still in flight (early loop exit) before the CTA may retire.
__device__ __forceinline__ void st_drain(Streamer& st) {
    for (uint64_t e = st.consumed; e < st.issued; ++e)
        mbar_wait(st.bars + e % st.ns, static_cast<unsigned>((e / st.ns) & 1u));
    st.consumed = st.issued;
}

// ---------------------------------------------------------------- estimate_step kernel
// Power iteration on P^-1/2 Theta^T Theta P^-1/2 (solver.cpp:69-99). The reference's
// v_k = w_k / |w_k| followed by u = P^-1/2 v is folded into the next product:
// Theta (P^-1/2 v_k) = (Theta (P^-1/2 w_k)) / |w_k|, so an iteration is two phases.
template <typename T>
__global__ void __launch_bounds__(kBlock, WBX_TAU_MINB) tau_kernel(SolveArgs a) {
    __shared__ double smem[kWarpsPerBlock + 1];
    const int lane = threadIdx.x & 31;
    const uint32_t gwarp = (blockIdx.x * kBlock + threadIdx.x) >> 5;
    const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kBlock;
    const unsigned epoch0 = *reinterpret_cast<volatile unsigned*>(a.sync.gen);
    Epoch epoch{epoch0, epoch0};
    extern __shared__ __align__(16) unsigned char dsmem[];
    Streamer st{};
    if constexpr (sizeof(T) == 4)
        st_init(st, dsmem + (threadIdx.x >> 5) * warp_smem_bytes(a.nslots), a.A, a.T, gwarp, nwarps, lane, 200,
                false, a.nslots);
    // row loop of one phase: TMA-staged fp32 operator with fp32 vectors (T = float, as in the
    // window engine) or the exact fp64 layout with fp64 vectors (T = double)
    using V = T;
    V* uC = sizeof(T) == 4 ? reinterpret_cast<V*>(a.yC) : reinterpret_cast<V*>(a.uC);   // P^-1/2 w on C
    V* tR = sizeof(T) == 4 ? reinterpret_cast<V*>(a.res) : reinterpret_cast<V*>(a.t64);  // Theta u on R
    auto phase = [&](bool isT, const V* x, auto pre, auto post) {
        if constexpr (sizeof(T) == 4)
            st_phase<float, float>(st, a.A, a.T, gwarp, nwarps, lane, isT ? st.nT : st.nA, x, pre, post);
        else
            for_rows_exact(isT ? a.T : a.A, gwarp, nwarps, lane, x,
                           [&](uint32_t r, double v) { post(r, v, pre(r)); });
    };

    // v0 = CounterRng(0x5eed) normals over ALL n, normalised by the full norm; only the
    // C part ever meets Theta (Theta^T output is zero outside C).
    double s2[1] = {0.0};
    for (uint64_t i = gthread; i < a.n; i += nthreads) {
        const double v = rng_normal(0x5eedull, i);
        s2[0] += v * v;
    }
    for (uint64_t c = gthread; c < a.nC; c += nthreads) {
        const double v = rng_normal(0x5eedull, a.C_glob[c]);
        a.wv[c] = v;                              // "w_prev" = raw v0, |w_prev| = |v0|
        uC[c] = static_cast<V>(a.ispC[c] * v);    // P^-1/2 w_prev
    }
    grid_sync_reduce<1>(a.sync, epoch, s2, smem);
    double nw_prev = sqrt(s2[0]);
    double lambda_prev = 0.0;
    int it = 0;
    bool zero_op = false;
    for (; it < 200; ++it) {
        // t = Theta (P^-1/2 v) = Theta (P^-1/2 w_prev) / |w_prev|
        const double inv = nw_prev;
        phase(
            false, uC, [](uint32_t) { return 0; },
            [&](uint32_t r, double t, int) { tR[r] = static_cast<V>(t / inv); });
        grid_sync(a.sync, epoch, smem);
        // w = P^-1/2 Theta^T t ; <v, w>, <w, w> with v = w_prev / |w_prev|
        double acc[2] = {0.0, 0.0};
        phase(
            true, tR,
            [&](uint32_t c) { return c != kNoRow ? make_double2(a.ispC[c], a.wv[c]) : make_double2(0.0, 0.0); },
            [&](uint32_t c, double g, double2 pv) {
                const double w = g * pv.x;
                const double v = pv.y / inv;
                acc[0] += v * w;
                acc[1] += w * w;
                a.wv[c] = w;
                uC[c] = static_cast<V>(pv.x * w);
            });
        grid_sync_reduce<2>(a.sync, epoch, acc, smem);
        const double lambda = acc[0];
        const double nw = sqrt(acc[1]);
        if (nw == 0.0) {  // zero operator sentinel (solver.cpp:89)
            zero_op = true;
            ++it;
            break;
        }
        if (it > 0 && fabs(lambda - lambda_prev) <= 1e-6 * fabs(lambda)) {
            lambda_prev = lambda;
            ++it;
            break;
        }
        lambda_prev = lambda;
        nw_prev = nw;
    }
    if constexpr (sizeof(T) == 4) st_drain(st);
    if (gthread == 0) {
        a.out[OUT_TAU] = (zero_op || lambda_prev <= 0.0) ? 1.0 : 1.0 / (lambda_prev * a.step_safety);
        a.out[OUT_TAU_ITERS] = it > 200 ? 200 : it;
        a.out[OUT_TAU_STEPS] = it > 200 ? 200 : it;
        a.out[OUT_LAMBDA_MAX] = lambda_prev;
    }
}

// ---------------------------------------------------------------- FISTA kernel
template <typename T>
__global__ void __launch_bounds__(kBlock, WBX_FISTA_MINB) fista_kernel(SolveArgs a) {
    __shared__ double smem[kWarpsPerBlock + 1];
    const int lane = threadIdx.x & 31;
    const uint32_t gwarp = (blockIdx.x * kBlock + threadIdx.x) >> 5;
    const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kBlock;
    const unsigned epoch0 = *reinterpret_cast<volatile unsigned*>(a.sync.gen);
    Epoch epoch{epoch0, epoch0};
    T* yC = static_cast<T*>(a.yC);
    T* xpC = static_cast<T*>(a.xpC);
    T* res = static_cast<T*>(a.res);
    T* x0R = static_cast<T*>(a.x0R);
    T* tpC = static_cast<T*>(a.tpC);
    T* thrC = static_cast<T*>(a.thrC);
    const Plan pA = sizeof(T) == 4 && a.track ? make_plan(a.A, gwarp, nwarps, lane) : Plan{};
    const double tau = a.tau_from_device ? a.out[OUT_TAU] : a.tau_given;
    extern __shared__ __align__(16) unsigned char dsmem[];
    Streamer st{};
    if constexpr (sizeof(T) == 4)
        st_init(st, dsmem + (threadIdx.x >> 5) * warp_smem_bytes(a.nslots), a.A, a.T, gwarp, nwarps, lane,
                static_cast<uint64_t>(a.max_iters), a.track != 0, a.nslots);
    auto phase = [&](bool isT, const T* x, auto pre, auto post) {
        if constexpr (sizeof(T) == 4)
            st_phase<float, float>(st, a.A, a.T, gwarp, nwarps, lane, isT ? st.nT : st.nA, x, pre, post);
        else
            for_rows_exact(isT ? a.T : a.A, gwarp, nwarps, lane, x, [&](uint32_t r, T v) { post(r, v, pre(r)); });
    };
    auto pre_x0 = [&](uint32_t r) { return r != kNoRow ? x0R[r] : T(0); };
    // epilogue operands of the fused update, loaded before the gathers
    struct Coord {
        T y, xp, tp, thr;
    };
    auto pre_coord = [&](uint32_t c) {
        Coord q{T(0), T(0), T(0), T(0)};
        if (c != kNoRow) {
            q.y = yC[c];
            q.xp = xpC[c];
            q.tp = tpC[c];
            q.thr = thrC[c];
        }
        return q;
    };

    // ---- init: compacted copies of x0; warm start x = x_prev = y = x0 (solver.cpp:115-117);
    // per-coordinate tau/p and tau*lambda*w/p on C
    for (uint64_t c = gthread; c < a.nC; c += nthreads) {
        const T v = static_cast<T>(a.x0_full[a.C_glob[c]]);
        yC[c] = v;
        xpC[c] = v;
        tpC[c] = static_cast<T>(tau / a.pC[c]);
        thrC[c] = static_cast<T>(thr_exact(tau, a.lambda, a.wC[c], a.pC[c]));
    }
    for (uint64_t r = gthread; r < a.nR; r += nthreads) x0R[r] = static_cast<T>(a.x0_full[a.R_glob[r]]);

    // ---- decoupled coordinates (independent of everything else)
    if (a.decoupled_inline) decoupled_pass<T>(a, tau, a.max_iters, 0, gthread, nthreads, nullptr, nullptr, 0);

    // ---- tracking: initial energy E(x0) (solver.cpp:118)
    double stop_gap = 0.0, quad_nonR = 0.0;
    if (a.track) {
        grid_sync(a.sync, epoch, smem);  // yC / x0R complete
        double e[3] = {0.0, 0.0, 0.0};
        for (uint64_t i = gthread; i < a.n; i += nthreads) {
            const double x0 = a.x0_full[i];
            if (!bit_set(a.isR, i)) e[0] += x0 * x0;
            e[1] += a.w_full[i] * fabs(x0);
        }
        for_rows<T, T, T>(a.A, pA, gwarp, nwarps, lane, yC, [&](uint32_t r, T t) {
            const double d = static_cast<double>(t) - static_cast<double>(x0R[r]);
            e[2] += d * d;
        });
        grid_sync_reduce<3>(a.sync, epoch, e, smem);
        quad_nonR = e[0];
        const double e0 = 0.5 * (e[2] + quad_nonR) + a.lambda * e[1];
        stop_gap = a.rel_tol * e0;
        if (gthread == 0) a.out[OUT_INITIAL_ENERGY] = e0;
    } else {
        grid_sync(a.sync, epoch, smem);
    }

    // ---- the FISTA / ISTA loop (solver.cpp:121-151)
    int k = 1;
    for (; k <= a.max_iters; ++k) {
        // phase A: res = Theta y - x0 on nonempty rows
        phase(false, yC, pre_x0, [&](uint32_t r, T acc, T x0) { res[r] = Prec<T>::sub(acc, x0); });
        grid_sync(a.sync, epoch, smem);
        // phase T: gradient on nonempty columns + fused step / prox / momentum
        const T beta = Prec<T>::beta(a, k);
        double tr[3] = {0.0, 0.0, 0.0};
        phase(true, res, pre_coord, [&](uint32_t c, T g, const Coord& q) {
            const T z0 = Prec<T>::z0(q.y, g, q.tp, tau, sizeof(T) == 8 ? a.pC[c] : 0.0);
            const T xn = Prec<T>::prox(z0, q.thr);
            yC[c] = Prec<T>::momentum(xn, q.xp, beta);
            xpC[c] = xn;
            if (a.track) {
                tr[1] += a.wC[c] * fabs(static_cast<double>(xn));
                tr[2] += xn != T(0) ? 1.0 : 0.0;
            }
        });
        grid_sync(a.sync, epoch, smem);
        if (a.track) {
            // energy(x') (solver.cpp:130, :44-55): Theta x' on rows R
            phase(false, xpC, pre_x0, [&](uint32_t r, T t, T x0) {
                const double d = static_cast<double>(t) - static_cast<double>(x0);
                tr[0] += d * d;
            });
            grid_sync_reduce<3>(a.sync, epoch, tr, smem);
            const double e = 0.5 * (tr[0] + quad_nonR) + a.lambda * (tr[1] + a.dec_reg[k - 1]);
            if (gthread == 0) {
                a.energies[k - 1] = e;
                a.supports[k - 1] = static_cast<unsigned long long>(tr[2] + a.dec_supp[k - 1]);
            }
            if (!isfinite(e)) {
                if (gthread == 0) a.out[OUT_STATUS] = 8.0;
                break;  // NonFiniteEnergy (solver.cpp:131-133); uniform across blocks
            }
            if (a.stop_on_ref && e - a.ref_energy <= stop_gap) {
                ++k;
                break;
            }
        }
    }
    if constexpr (sizeof(T) == 4) st_drain(st);
    const int used = k - 1 > a.max_iters ? a.max_iters : k - 1;
    if (gthread == 0) a.out[OUT_ITERS_USED] = used;
    // ---- x_final on C back into the full coefficient vector
    for (uint64_t c = gthread; c < a.nC; c += nthreads) a.x_full[a.C_glob[c]] = static_cast<double>(xpC[c]);
}

// ---------------------------------------------------------------- window engine (win.cuh)
// CTA size of the window engine (WBX_WIN_BLOCK=512: one CTA per SM, experiment)
#ifndef WBX_WIN_BLOCK
#define WBX_WIN_BLOCK 256
#endif
constexpr int kWinBlock = WBX_WIN_BLOCK;
constexpr int kWinWarps = kWinBlock / 32;
#ifndef WBX_WIN_MINB
#define WBX_WIN_MINB (512 / WBX_WIN_BLOCK)
#endif
constexpr int kWinMinBlocks = WBX_WIN_MINB;  // CTAs per SM the window kernels are built for
// Shared memory of a CTA:
//   [uA][uT]          window index lists of the two sides              } loaded once
//   [sA][sT]          slice tables {record offset, meta, first row}    } per solve
//   [dA][dT]          value dictionaries (dictionary format)           }
//   [own A][own T]    per-row state of the CTA's own contiguous row ranges (e.g. y, x_prev,
//                     tau/p, threshold of its coordinates): only this CTA updates those rows,
//                     so the state lives on chip for the whole solve
//   [window]          x[U_b] of the current phase
__host__ __device__ constexpr uint32_t win_align16(uint32_t b) { return (b + 15u) & ~15u; }

struct WinSmem {
    uint32_t* uA;
    uint32_t* uT;
    uint16_t* usA;  // window slot of each entry
    uint16_t* usT;
    uint4* sA;
    uint4* sT;
    float* dA;
    float* dT;
    void* ownA;
    void* ownT;
    void* win;
    uint32_t nuA, nuT, nsA, nsT;
    uint32_t rA0, rT0, nrA, nrT;  // own row ranges
};

// lists_global: the window index lists (entries and slots) stay in global memory (L2) and are
// read by the fill itself — for operators whose windows are too large for both lists and
// window in shared memory (the spatially varying C3 operator at 1024^2)
template <uint32_t OWN_A, uint32_t OWN_T>
__host__ __device__ inline uint32_t win_smem_head(const WinView& A, const WinView& T, bool lists_global = false) {
    const uint32_t lists = lists_global ? 0u
                                        : win_align16(A.max_u * 4u) + win_align16(T.max_u * 4u) +
                                              win_align16(A.max_u * 2u) + win_align16(T.max_u * 2u);
    return lists + 16u * (A.max_slices + T.max_slices) +
           win_align16(A.max_dict * 4u) + win_align16(T.max_dict * 4u) + win_align16(A.max_rows * OWN_A) +
           win_align16(T.max_rows * OWN_T);
}

template <uint32_t OWN_A, uint32_t OWN_T, bool LG>
__device__ __forceinline__ WinSmem win_smem_init(unsigned char* base, const SolveArgs& a) {
    WinSmem w;
    const uint32_t b = blockIdx.x;
    w.nuA = a.wA.u_off[b + 1] - a.wA.u_off[b];
    w.nuT = a.wT.u_off[b + 1] - a.wT.u_off[b];
    w.nsA = a.wA.s_off[b + 1] - a.wA.s_off[b];
    w.nsT = a.wT.s_off[b + 1] - a.wT.s_off[b];
    w.rA0 = a.wA.r_off[b];
    w.rT0 = a.wT.r_off[b];
    w.nrA = a.wA.r_off[b + 1] - w.rA0;
    w.nrT = a.wT.r_off[b + 1] - w.rT0;
    unsigned char* p = base;
    auto carve = [&](uint32_t bytes) {
        unsigned char* q = p;
        p += bytes;
        return q;
    };
    if (LG) {  // read in place by the fills (never written)
        w.uA = const_cast<uint32_t*>(a.wA.u_idx + a.wA.u_off[b]);
        w.uT = const_cast<uint32_t*>(a.wT.u_idx + a.wT.u_off[b]);
        w.usA = const_cast<uint16_t*>(a.wA.u_slot + a.wA.u_off[b]);
        w.usT = const_cast<uint16_t*>(a.wT.u_slot + a.wT.u_off[b]);
    } else {
        w.uA = reinterpret_cast<uint32_t*>(carve(win_align16(a.wA.max_u * 4u)));
        w.uT = reinterpret_cast<uint32_t*>(carve(win_align16(a.wT.max_u * 4u)));
        w.usA = reinterpret_cast<uint16_t*>(carve(win_align16(a.wA.max_u * 2u)));
        w.usT = reinterpret_cast<uint16_t*>(carve(win_align16(a.wT.max_u * 2u)));
    }
    w.sA = reinterpret_cast<uint4*>(carve(16u * a.wA.max_slices));
    w.sT = reinterpret_cast<uint4*>(carve(16u * a.wT.max_slices));
    w.dA = reinterpret_cast<float*>(carve(win_align16(a.wA.max_dict * 4u)));
    w.dT = reinterpret_cast<float*>(carve(win_align16(a.wT.max_dict * 4u)));
    w.ownA = carve(win_align16(a.wA.max_rows * OWN_A));
    w.ownT = carve(win_align16(a.wT.max_rows * OWN_T));
    w.win = p;
    if (!LG) {
        for (uint32_t i = threadIdx.x; i < w.nuA; i += kWinBlock) w.uA[i] = a.wA.u_idx[a.wA.u_off[b] + i];
        for (uint32_t i = threadIdx.x; i < w.nuT; i += kWinBlock) w.uT[i] = a.wT.u_idx[a.wT.u_off[b] + i];
        for (uint32_t i = threadIdx.x; i < w.nuA; i += kWinBlock) w.usA[i] = a.wA.u_slot[a.wA.u_off[b] + i];
        for (uint32_t i = threadIdx.x; i < w.nuT; i += kWinBlock) w.usT[i] = a.wT.u_slot[a.wT.u_off[b] + i];
    }
    for (uint32_t i = threadIdx.x; i < w.nsA; i += kWinBlock) w.sA[i] = a.wA.s_tab[a.wA.s_off[b] + i];
    for (uint32_t i = threadIdx.x; i < w.nsT; i += kWinBlock) w.sT[i] = a.wT.s_tab[a.wT.s_off[b] + i];
    if (a.wA.max_dict)
        for (uint32_t i = a.wA.d_off[b] + threadIdx.x; i < a.wA.d_off[b + 1]; i += kWinBlock)
            w.dA[i - a.wA.d_off[b]] = a.wA.d_val[i];
    if (a.wT.max_dict)
        for (uint32_t i = a.wT.d_off[b] + threadIdx.x; i < a.wT.d_off[b + 1]; i += kWinBlock)
            w.dT[i - a.wT.d_off[b]] = a.wT.d_val[i];
    __syncthreads();
    return w;
}

// One lane's share of a slice record in registers: dictionary offset (dictionary format)
// or values (full format), and up to 4 quads of 16-bit window columns.
template <bool DICT>
struct WinSlice {
    uint32_t pb;
    uint4 v[DICT ? 1 : 4];
    uint2 c[4];
};

template <bool DICT>
__device__ __forceinline__ void win_load(const uint4* rec_base, const uint4& sl, int lane, uint64_t pol,
                                         WinSlice<DICT>& d) {
    const uint4* rec = rec_base + sl.x;
    const int nq = static_cast<int>(sl.y & 0xffu);
    const uint2* cols = reinterpret_cast<const uint2*>(rec + (DICT ? 4 : nq * 32));
    if (DICT) d.pb = ld_stream(reinterpret_cast<const uint16_t*>(rec) + lane, pol);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (!DICT) d.v[q] = q < nq ? ld_stream(rec + q * 32 + lane, pol) : make_uint4(0, 0, 0, 0);
        d.c[q] = q < nq ? ld_stream(cols + q * 32 + lane, pol) : make_uint2(0, 0);
    }
}

// WBX_PROFILE=3: per-warp cycle accounting of the window engine (wbx_diag_slice_profile)
struct WinProf {
    // [A fill, A slice loop, A barrier, T fill, T slice loop, T barrier, -, -] (cycles, summed)
    unsigned long long c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int side = 0;  // 0 = phase A, 3 = phase T (set before each phase, used by the timers)
    __device__ __forceinline__ void flush() {
        if (WBX_PROFILE == 3 && (threadIdx.x & 31) == 0)
            for (int i = 0; i < 8; ++i) atomicAdd(&g_prof[i], c[i]);
    }
};

// One phase on the window engine: fill the CTA's window from x (asynchronous copies, one
// parallel round trip; the first slices' record loads are issued before it since they do
// not depend on x), then every warp runs its slices (w, w+8, ...) with one slice of
// record loads in flight; the vector operand and (dictionary format) the values come from
// shared memory.
struct NoHook {
    __device__ void operator()() const {}
};

template <typename ACC, typename WIN, bool DICT, typename X, typename Post, typename Ready = NoHook>
__device__ __forceinline__ void win_phase(const WinView& W, const uint32_t* uidx, const uint16_t* uslot, uint32_t nu,
                                          const uint4* stab,
                                          uint32_t ns, const float* dict, const X* __restrict__ x, WIN* win,
                                          Post post, WinProf& pf, Ready ready = Ready{}) {
    static_assert(sizeof(WIN) == sizeof(X), "the window is a verbatim copy of x entries");
    const long long t0 = WBX_PROFILE == 3 ? clock64() : 0;
    const int lane = threadIdx.x & 31;
    const uint32_t wib = threadIdx.x >> 5;
    const uint64_t pol = l2_keep_policy();
    WinSlice<DICT> b0, b1;
    if (wib < ns) win_load<DICT>(W.rec, stab[wib], lane, pol, b0);
    // window fill (L1 lines are invalidated by the grid barrier's acquire)
    if (sizeof(X) == 4 && W.chunk) {  // chunk layout: 16-byte copies, chunk i to window floats 4 slot(i)..
        for (uint32_t i = threadIdx.x; i < nu; i += kWinBlock) {
            WBX_ASSERT(4u * uslot[i] + 3 < W.max_win && 4 * uidx[i] < W.src_len);
            const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(win + 4u * uslot[i]));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(x + 4 * uidx[i]) : "memory");
        }
    } else {
        for (uint32_t i = threadIdx.x; i < nu; i += kWinBlock) {
            WBX_ASSERT(uslot[i] < W.max_win && uidx[i] < W.src_len);
            const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(win + uslot[i]));
            asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst), "l"(x + uidx[i]), "n"(sizeof(X))
                         : "memory");
        }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    ready();  // every copy issued before the phase (window, staged partials) has landed
    const long long t1 = WBX_PROFILE == 3 ? clock64() : 0;
    // process slice s from d
    // dictionary values of the lane's last segment block: consecutive slices of a warp are
    // mostly the same band rows at the same positions, so a lane's block rarely changes and
    // the reload (4 x LDS.128) is skipped
    uint32_t cpb = 0xffffffffu;
    float4 cv[4];
    auto run = [&](const WinSlice<DICT>& d, uint32_t s) {
        const uint4 sl = stab[s];  // {record offset, meta, first row, -}
        const uint32_t nq = sl.y & 0xffu, m = (sl.y >> 8) & 0xffu, nseg = (sl.y >> 16) & 0xffu;
        const uint32_t cnt = sl.y >> 24;
        WBX_ASSERT(s < ns && nq >= 1 && nq <= 4 && m >= 1 && m * nseg <= 32 && cnt <= m);
        WBX_ASSERT(!DICT || d.pb + 15 < W.max_dict);
        if (DICT && WBX_DICT_CACHE && d.pb != cpb) {
            cpb = d.pb;
#pragma unroll
            for (uint32_t qd = 0; qd < 4; ++qd) cv[qd] = *reinterpret_cast<const float4*>(dict + cpb + qd * 4);
        }
        ACC acc = ACC(0);
#pragma unroll
        for (uint32_t qd = 0; qd < 4; ++qd) {
            if (qd < nq) {
                float4 v;
                if (DICT) {
                    v = WBX_DICT_CACHE ? cv[qd] : *reinterpret_cast<const float4*>(dict + d.pb + qd * 4);
                } else {
                    v = make_float4(__uint_as_float(d.v[qd].x), __uint_as_float(d.v[qd].y),
                                    __uint_as_float(d.v[qd].z), __uint_as_float(d.v[qd].w));
                }
                WBX_ASSERT((d.c[qd].x & 0xffffu) < W.max_win && (d.c[qd].x >> 16) < W.max_win &&
                           (d.c[qd].y & 0xffffu) < W.max_win && (d.c[qd].y >> 16) < W.max_win);
                const WIN g0 = win[d.c[qd].x & 0xffffu], g1 = win[d.c[qd].x >> 16];
                const WIN g2 = win[d.c[qd].y & 0xffffu], g3 = win[d.c[qd].y >> 16];
                acc = fma(static_cast<ACC>(v.x), static_cast<ACC>(g0), acc);
                acc = fma(static_cast<ACC>(v.y), static_cast<ACC>(g1), acc);
                acc = fma(static_cast<ACC>(v.z), static_cast<ACC>(g2), acc);
                acc = fma(static_cast<ACC>(v.w), static_cast<ACC>(g3), acc);
            }
        }
        // segments of row i sit in lanes i, i+m, ..., i+(nseg-1)m: fold into the head lane
        for (uint32_t t = 1; t < nseg; ++t) {
            const ACC o = __shfl_down_sync(0xffffffffu, acc, t * m);
            if (static_cast<uint32_t>(lane) < m) acc += o;
        }
        if (static_cast<uint32_t>(lane) < cnt) post(sl.z + lane, acc);
    };
    // one slice of record loads in flight: the next load is issued before the current slice
    // computes (deeper lookahead and paired slices measured slower: register pressure)
    for (uint32_t s = wib; s < ns; s += kWinWarps) {
        b1 = b0;
        if (s + kWinWarps < ns) win_load<DICT>(W.rec, stab[s + kWinWarps], lane, pol, b0);
        run(b1, s);
    }
    if (WBX_PROFILE == 3) {
        const long long t2 = clock64();
        pf.c[pf.side] += t1 - t0;
        pf.c[pf.side + 1] += t2 - t1;
    }
    __syncthreads();  // the window is refilled by the next phase
}

template <bool DICT, bool LG>
__global__ void __launch_bounds__(kWinBlock, kWinMinBlocks) fista_win_kernel(SolveArgs a) {
    __shared__ double smem[kWinWarps + 1];
    extern __shared__ __align__(16) unsigned char dsmem[];
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kWinBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kWinBlock;
    const unsigned epoch0 = *reinterpret_cast<volatile unsigned*>(a.sync.gen);
    Epoch epoch{epoch0, epoch0};
    float* yC = static_cast<float*>(a.yC);
    float* res = static_cast<float*>(a.res);
    const double tau = a.tau_from_device ? a.out[OUT_TAU] : a.tau_given;
    const WinSmem ws = win_smem_init<4, 16, LG>(dsmem, a);
    float* win = static_cast<float*>(ws.win);
    float* x0s = static_cast<float*>(ws.ownA);   // x0 of the CTA's Theta rows
    float4* cs = static_cast<float4*>(ws.ownT);  // {y, x_prev, tau/p, threshold} of its coordinates
    for (uint32_t i = threadIdx.x; i < ws.nrT; i += kWinBlock) {
        const uint32_t c = ws.rT0 + i;
        const float v = static_cast<float>(a.x0_full[a.C_glob[c]]);
        yC[c] = v;
        cs[i] = make_float4(v, v, static_cast<float>(tau / a.pC[c]),
                            static_cast<float>(thr_exact(tau, a.lambda, a.wC[c], a.pC[c])));
    }
    for (uint32_t i = threadIdx.x; i < ws.nrA; i += kWinBlock)
        x0s[i] = static_cast<float>(a.x0_full[a.R_glob[ws.rA0 + i]]);
    if (a.decoupled_inline) decoupled_pass<float>(a, tau, a.max_iters, 0, gthread, nthreads, nullptr, nullptr, 0);
    grid_sync(a.sync, epoch, smem);
    WinProf pf;
    auto sync = [&]() {
        const long long b0 = WBX_PROFILE == 3 ? clock64() : 0;
        grid_sync(a.sync, epoch, smem);
        if (WBX_PROFILE == 3) pf.c[pf.side + 2] += clock64() - b0;
    };
    for (int k = 1; k <= a.max_iters; ++k) {
        pf.side = 0;
        win_phase<float, float, DICT>(a.wA, ws.uA, ws.usA, ws.nuA, ws.sA, ws.nsA, ws.dA, yC, win,
                                          [&](uint32_t r, float acc) {
                                              WBX_ASSERT(r - ws.rA0 < ws.nrA);
                                              res[r] = acc - x0s[r - ws.rA0];
                                          }, pf);
        sync();
        const float beta = a.beta32[k - 1];
        pf.side = 3;
        win_phase<float, float, DICT>(a.wT, ws.uT, ws.usT, ws.nuT, ws.sT, ws.nsT, ws.dT, res, win,
                                          [&](uint32_t c, float g) {
                                              WBX_ASSERT(c - ws.rT0 < ws.nrT);
                                              float4& s = cs[c - ws.rT0];
                                              const float z0 = fmaf(-s.z, g, s.x);
                                              const float xn = Prec<float>::prox(z0, s.w);
                                              const float yn = fmaf(beta, xn - s.y, xn);
                                              s.x = yn;
                                              s.y = xn;
                                              yC[c] = yn;
                                          },
                                          pf);
        sync();
    }
    pf.flush();
    if (gthread == 0) a.out[OUT_ITERS_USED] = a.max_iters;
    for (uint32_t i = threadIdx.x; i < ws.nrT; i += kWinBlock) a.x_full[a.C_glob[ws.rT0 + i]] = static_cast<double>(cs[i].y);
}

// Sum of three sets of G per-CTA partials in a fixed order (identical in every CTA); all threads.
__device__ __forceinline__ void cta_sum3(const double* p0, const double* p1, const double* p2, unsigned G,
                                         double* red3, double (&out)[3]) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (unsigned i = threadIdx.x; i < G; i += kWinBlock) {
        s0 += p0[i];
        s1 += p1[i];
        s2 += p2[i];
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if ((threadIdx.x & 31) == 0) {
        red3[3 * (threadIdx.x >> 5) + 0] = s0;
        red3[3 * (threadIdx.x >> 5) + 1] = s1;
        red3[3 * (threadIdx.x >> 5) + 2] = s2;
    }
    __syncthreads();
    out[0] = out[1] = out[2] = 0.0;
#pragma unroll
    for (int k = 0; k < kWinWarps; ++k) {
        out[0] += red3[3 * k + 0];
        out[1] += red3[3 * k + 1];
        out[2] += red3[3 * k + 2];
    }
    __syncthreads();
}

// block partial (fixed tree) of v -> dst[blockIdx.x]; all threads
__device__ __forceinline__ void win_block_partial(double v, double* dst, double* red) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < kWinWarps; ++k) t += red[k];
        dst[blockIdx.x] = t;
    }
    __syncthreads();
}

// FISTA / ISTA on the window engine WITH the reference's per-iteration bookkeeping
// (run_pgd, solver.cpp:118-150): E(x_0), E(x_k) and the support size every iteration, the
// NonFiniteEnergy check and the ref_energy stopping rule — still two operator products per
// iteration. The reference spends a third SpMV on energy(x_k) (Theta x_k, solver.cpp:44-55);
// here Theta x_k comes by linearity from the phase-A product of the next iteration:
//   y_k = x_k + beta_k (x_k - x_k-1)  =>  Theta x_k = (Theta y_k + beta_k Theta x_k-1) / (1 + beta_k),
// kept per own row of Theta in shared memory (u, next to x0). So E(x_k) is complete after phase
// A of iteration k+1 (one phase later): the stopping decision is taken there, before phase T
// overwrites x_k (x_prev in the CTA state). Every CTA sums the same per-CTA partials in the
// same order, so all take the same decision without further communication.
// Decoupled coordinates (empty Theta column) are tracked by decoupled_kernel (dec_reg/dec_supp).
template <bool DICT, bool LG>
__global__ void __launch_bounds__(kWinBlock, kWinMinBlocks) fista_win_track_kernel(SolveArgs a) {
    __shared__ double smem[kWinWarps + 1];
    __shared__ double red[3 * kWinWarps];
    extern __shared__ __align__(16) unsigned char dsmem[];
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kWinBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kWinBlock;
    const unsigned G = gridDim.x;
    const unsigned epoch0 = *reinterpret_cast<volatile unsigned*>(a.sync.gen);
    Epoch epoch{epoch0, epoch0};
    float* yC = static_cast<float*>(a.yC);
    float* res = static_cast<float*>(a.res);
    const double tau = a.tau_from_device ? a.out[OUT_TAU] : a.tau_given;
    const WinSmem ws = win_smem_init<8, 16, LG>(dsmem, a);
    float* win = static_cast<float*>(ws.win);
    float2* ra = static_cast<float2*>(ws.ownA);  // {x0, Theta x_k-1} of the CTA's Theta rows
    float4* cs = static_cast<float4*>(ws.ownT);  // {y, x_prev, tau/p, threshold} of its coordinates
    for (uint32_t i = threadIdx.x; i < ws.nrT; i += kWinBlock) {
        const uint32_t c = ws.rT0 + i;
        const float v = static_cast<float>(a.x0_full[a.C_glob[c]]);
        yC[c] = v;
        cs[i] = make_float4(v, v, static_cast<float>(tau / a.pC[c]),
                            static_cast<float>(thr_exact(tau, a.lambda, a.wC[c], a.pC[c])));
    }
    for (uint32_t i = threadIdx.x; i < ws.nrA; i += kWinBlock)
        ra[i] = make_float2(static_cast<float>(a.x0_full[a.R_glob[ws.rA0 + i]]), 0.f);
    // constant parts of the energy: sum of x0^2 over rows outside R (Theta x is 0 there) and
    // lambda-free sum of w |x0| over every coordinate (E(x_0))
    double e0s[2] = {0.0, 0.0};
    for (uint64_t i = gthread; i < a.n; i += nthreads) {
        const double x0 = a.x0_full[i];
        if (!bit_set(a.isR, i)) e0s[0] += x0 * x0;
        e0s[1] += a.w_full[i] * fabs(x0);
    }
    grid_sync_reduce<2, kWinBlock>(a.sync, epoch, e0s, smem);  // (also: yC complete)
    const double quad_nonR = e0s[0];
    double stop_gap = 0.0;
    // per-CTA partials, after the barrier-reduction slots (which other CTAs may still be reading
    // when a fast CTA starts phase A): [G] quadratic part of phase A; [2][G] w|x| and support of
    // phase T, double-buffered by iteration parity (read after the next A barrier)
    double* const tp = a.sync.part + static_cast<uint64_t>(2 * kRedSlots) * G;
    double* const q_part = tp;
    auto reg_part = [&](int k) { return tp + static_cast<uint64_t>(1 + 2 * (k & 1)) * G; };
    auto sup_part = [&](int k) { return tp + static_cast<uint64_t>(2 + 2 * (k & 1)) * G; };
    WinProf pf;
    int used = 0;
    for (int k = 1;; ++k) {
        // phase A of iteration k: res = Theta y_k-1 - x0; Theta x_k-1 by linearity
        const float bp = k >= 2 ? a.beta32[k - 2] : 0.f;  // beta_k-1
        const float inv = 1.f / (1.f + bp);
        double q = 0.0;
        win_phase<float, float, DICT>(a.wA, ws.uA, ws.usA, ws.nuA, ws.sA, ws.nsA, ws.dA, yC, win,
                                      [&](uint32_t r, float acc) {
                                          float2& st = ra[r - ws.rA0];
                                          res[r] = acc - st.x;
                                          const float u = k == 1 ? acc : fmaf(bp, st.y, acc) * inv;
                                          st.y = u;
                                          const double d = static_cast<double>(u) - static_cast<double>(st.x);
                                          q += d * d;
                                      },
                                      pf);
        win_block_partial(q, q_part, red);
        grid_sync(a.sync, epoch, smem);
        // E(x_k-1) (solver.cpp:44-55, 118, 130): quadratic part of this phase, weighted l1 and
        // support of phase T of iteration k-1 (+ the decoupled coordinates)
        double t[3];
        cta_sum3(q_part, reg_part(k - 1), sup_part(k - 1), G, red, t);
        if (k == 1) {
            const double e0 = 0.5 * (t[0] + quad_nonR) + a.lambda * e0s[1];
            stop_gap = a.rel_tol * e0;
            if (gthread == 0) a.out[OUT_INITIAL_ENERGY] = e0;
        } else {
            const double e = 0.5 * (t[0] + quad_nonR) + a.lambda * (t[1] + a.dec_reg[k - 2]);
            if (gthread == 0) {
                a.energies[k - 2] = e;
                a.supports[k - 2] = static_cast<unsigned long long>(t[2] + a.dec_supp[k - 2]);
            }
            used = k - 1;
            if (!isfinite(e)) {
                if (gthread == 0) a.out[OUT_STATUS] = 8.0;  // NonFiniteEnergy (solver.cpp:131-133)
                break;
            }
            if (a.stop_on_ref && e - a.ref_energy <= stop_gap) break;  // solver.cpp:150
        }
        if (k > a.max_iters) break;
        // phase T of iteration k: gradient + step + prox + momentum; sums of w|x_k|, support
        const float beta = a.beta32[k - 1];
        double rg = 0.0, sp = 0.0;
        win_phase<float, float, DICT>(a.wT, ws.uT, ws.usT, ws.nuT, ws.sT, ws.nsT, ws.dT, res, win,
                                      [&](uint32_t c, float g) {
                                          float4& s = cs[c - ws.rT0];
                                          const float z0 = fmaf(-s.z, g, s.x);
                                          const float xn = Prec<float>::prox(z0, s.w);
                                          const float yn = fmaf(beta, xn - s.y, xn);
                                          s.x = yn;
                                          s.y = xn;
                                          yC[c] = yn;
                                          rg += a.wC[c] * fabs(static_cast<double>(xn));
                                          sp += xn != 0.f ? 1.0 : 0.0;
                                      },
                                      pf);
        win_block_partial(rg, reg_part(k), red);
        win_block_partial(sp, sup_part(k), red);
        grid_sync(a.sync, epoch, smem);
    }
    pf.flush();
    if (gthread == 0) a.out[OUT_ITERS_USED] = used;
    for (uint32_t i = threadIdx.x; i < ws.nrT; i += kWinBlock) a.x_full[a.C_glob[ws.rT0 + i]] = static_cast<double>(cs[i].y);
}

// estimate_step on the window engine: fp64 accumulation, own state and reductions; fp32
// operator values; vector windows in WINT (float: the gathered u and t entries are rounded
// to fp32, the products are exact in fp64; double: fp64 windows, WBX_TAU_WINDOW=64)
template <bool DICT, typename WINT, bool LG>
__global__ void __launch_bounds__(kWinBlock, kWinMinBlocks) tau_win_kernel(SolveArgs a) {
    __shared__ double smem[kWinWarps + 1];
    extern __shared__ __align__(16) unsigned char dsmem[];
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kWinBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kWinBlock;
    const unsigned epoch0 = *reinterpret_cast<volatile unsigned*>(a.sync.gen);
    Epoch epoch{epoch0, epoch0};
    const WinSmem ws = win_smem_init<0, 16, LG>(dsmem, a);
    WINT* win = static_cast<WINT*>(ws.win);
    double2* cs = static_cast<double2*>(ws.ownT);  // {P^-1/2, w} of the CTA's coordinates
    constexpr bool W64 = sizeof(WINT) == 8;
    // row sums of the fp32 windows in fp32 (their inputs and outputs are fp32 already; the
    // Rayleigh-quotient partial sums stay fp64); WBX_TAU_ACC32=0 accumulates in fp64
    using TACC = typename std::conditional<WBX_TAU_ACC32 && !W64, float, double>::type;
    WINT* uC = W64 ? reinterpret_cast<WINT*>(a.uC) : static_cast<WINT*>(a.yC);  // u = P^-1/2 w on C
    WINT* tR = W64 ? reinterpret_cast<WINT*>(a.t64) : static_cast<WINT*>(a.res);  // t = Theta u on R
    double s2[1] = {0.0};
    for (uint64_t i = gthread; i < a.n; i += nthreads) {
        const double v = rng_normal(0x5eedull, i);
        s2[0] += v * v;
    }
    for (uint32_t i = threadIdx.x; i < ws.nrT; i += kWinBlock) {
        const uint32_t c = ws.rT0 + i;
        const double v = rng_normal(0x5eedull, a.C_glob[c]);
        const double isp = a.ispC[c];
        cs[i] = make_double2(isp, v);
        uC[c] = static_cast<WINT>(isp * v);
    }
    grid_sync_reduce<1, kWinBlock>(a.sync, epoch, s2, smem);
    double nw_prev = sqrt(s2[0]);
    double lambda_prev = 0.0;
    int it = 0, iters = 0;
    bool zero_op = false;
    WinProf pf;
    __shared__ double red[2];
    const unsigned G = gridDim.x;
    // staging of the 2 x G block partials, after the window
    double* pstage = reinterpret_cast<double*>(
        static_cast<unsigned char*>(ws.win) + win_align16((a.wA.max_win > a.wT.max_win ? a.wA.max_win : a.wT.max_win) * sizeof(WINT)));
    // Deferred reduction: phase A computes Theta u WITHOUT the 1/|w_prev| normalisation (it is
    // applied to Theta^T t in phase T instead), so A does not wait for the previous
    // iteration's grid reduction; the block partials of iteration it-1 are summed by warp 0
    // while phase A of iteration it runs, and its stopping test is taken after A. Every
    // barrier is a plain one. (On convergence one extra phase A has been computed.)
    for (it = 0;; ++it) {
        const double* part = a.sync.part + static_cast<uint64_t>((it + 1) & 1) * kRedSlots * G;
        if (it > 0 && threadIdx.x < 32)  // asynchronous copies, complete during the phase
            for (unsigned i = threadIdx.x; i < 2 * G; i += 32) {
                const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(pstage + i));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst),
                             "l"(part + i) : "memory");
            }
        pf.side = 0;
        if (it < 200)
            win_phase<TACC, WINT, DICT>(a.wA, ws.uA, ws.usA, ws.nuA, ws.sA, ws.nsA, ws.dA, uC, win,
                                              [&](uint32_t r, double t) { tR[r] = static_cast<WINT>(t); }, pf);
        if (it > 0) {  // the whole CTA sums the staged partials (fixed order, same in every CTA)
            if (it == 200) {  // no phase A ran: wait for the staging copies here
                asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
                __syncthreads();
            }
            __shared__ double2 ps[kWinWarps];
            double p0 = 0.0, p1 = 0.0;
            for (unsigned i = threadIdx.x; i < G; i += kWinBlock) {
                p0 += pstage[i];
                p1 += pstage[G + i];
            }
            p0 = warp_sum(p0);
            p1 = warp_sum(p1);
            if ((threadIdx.x & 31) == 0) ps[threadIdx.x >> 5] = make_double2(p0, p1);
            __syncthreads();
            if (threadIdx.x == 0) {
                double t0 = 0.0, t1 = 0.0;
                for (int k = 0; k < kWinWarps; ++k) {
                    t0 += ps[k].x;
                    t1 += ps[k].y;
                }
                red[0] = t0;
                red[1] = t1;
            }
        }
        const long long b0 = WBX_PROFILE == 3 ? clock64() : 0;
        grid_sync(a.sync, epoch, smem);
        if (WBX_PROFILE == 3) pf.c[pf.side + 2] += clock64() - b0;
        if (it > 0) {  // stopping test of iteration it-1 (solver.cpp:84-88)
            const double lambda = red[0];
            const double nw = sqrt(red[1]);
            if (nw == 0.0) {
                zero_op = true;
                iters = it;
                break;
            }
            if (it > 1 && fabs(lambda - lambda_prev) <= 1e-6 * fabs(lambda)) {
                lambda_prev = lambda;
                iters = it;
                break;
            }
            lambda_prev = lambda;
            nw_prev = nw;
        }
        if (it == 200) {
            iters = 200;
            break;
        }
        const double rinv = 1.0 / nw_prev;
        double acc[2] = {0.0, 0.0};
        pf.side = 3;
        win_phase<TACC, WINT, DICT>(a.wT, ws.uT, ws.usT, ws.nuT, ws.sT, ws.nsT, ws.dT, tR, win,
                                            [&](uint32_t c, double g) {
                                                WBX_ASSERT(c - ws.rT0 < ws.nrT);
                                                double2& s = cs[c - ws.rT0];
                                                const double w = (g * rinv) * s.x;
                                                const double v = s.y * rinv;
                                                acc[0] += v * w;
                                                acc[1] += w * w;
                                                s.y = w;
                                                uC[c] = static_cast<WINT>(s.x * w);
                                            },
                                            pf);
        double* wpart = a.sync.part + static_cast<uint64_t>(it & 1) * kRedSlots * G;
        {  // block partials of both sums, one fixed tree
            __shared__ double2 bs[kWinWarps];
            const double s0 = warp_sum(acc[0]), s1 = warp_sum(acc[1]);
            if ((threadIdx.x & 31) == 0) bs[threadIdx.x >> 5] = make_double2(s0, s1);
            __syncthreads();
            if (threadIdx.x == 0) {
                double t0 = 0.0, t1 = 0.0;
                for (int k = 0; k < kWinWarps; ++k) {
                    t0 += bs[k].x;
                    t1 += bs[k].y;
                }
                wpart[blockIdx.x] = t0;
                wpart[G + blockIdx.x] = t1;
            }
        }
        const long long b1 = WBX_PROFILE == 3 ? clock64() : 0;
        grid_sync(a.sync, epoch, smem);
        if (WBX_PROFILE == 3) pf.c[pf.side + 2] += clock64() - b1;
    }
    it = iters;
    pf.flush();
    if (gthread == 0) {
        a.out[OUT_TAU] = (zero_op || lambda_prev <= 0.0) ? 1.0 : 1.0 / (lambda_prev * a.step_safety);
        a.out[OUT_TAU_ITERS] = it > 200 ? 200 : it;
        a.out[OUT_TAU_STEPS] = it > 200 ? 200 : it;
        a.out[OUT_LAMBDA_MAX] = lambda_prev;
    }
}

// ---------------------------------------------------------------- estimate_step by Lanczos
// Window engine, fp32 hot path (WBX_TAU=power keeps tau_win_kernel; the fp64 mode keeps the
// literal power iteration).
//
// estimate_step (solver.cpp:69-99) runs the power iteration lambda_it = <v_it, M v_it>,
// v_it = M^it v0 / |M^it v0|, M = P^-1/2 Theta^T Theta P^-1/2, it < 200, and stops at the first
// it > 0 with |lambda_it - lambda_it-1| <= 1e-6 |lambda_it|. With mu_p = v0^T M^p v0 / |v0|^2,
// lambda_it = mu_{2it+1} / mu_{2it}. m Lanczos steps from v0 give the tridiagonal T_m with
// e1^T T_m^p e1 |v0_C|^2 / |v0|^2 = mu_p (p >= 1; v0_C = the part of v0 on Theta's nonempty
// columns) for every p <= 2m - 1 (Gauss quadrature). So the power iteration run on T_m from
// e1 reproduces the reference's lambda sequence, its stopping decision and tau. A Lanczos
// step costs the same two operator products as a power iteration, but the quadrature
// converges super-geometrically in m: at C2, estimates from successive m agree to 1e-15
// from m = 56 on, where the power iteration needs all 200 iterations. The kernel checks at
// m = lz_first (48), lz_first + lz_every, ... and stops once the estimates from T_m and
// T_{m-4} agree to lz_tol (1e-8) with the same stopping index, or at m = 200, where the
// identity covers every p <= 399 the reference can reach. The accepted estimate is much closer
// to the converged one than the bound (super-geometric convergence: at C2 T_48 is 1.4e-10 from
// T_60), below the fp32 rounding of tau/p the iterations use and the 2e-8 the fp32 operator
// values already move tau from the reference's; at C2 the estimate stops at m = 48 instead of
// 60 (tools/lz_sweep.py).
// sum of G staged block partials in a fixed order (the same in every CTA); all threads
__device__ __forceinline__ double cta_sum_staged(const double* st, unsigned G, double* red) {
    double p = 0.0;
    for (unsigned i = threadIdx.x; i < G; i += kWinBlock) p += st[i];
    p = warp_sum(p);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = p;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < kWinWarps; ++k) t += red[k];
    __syncthreads();
    return t;
}

__device__ __forceinline__ void stage_partials(double* dst, const double* src, unsigned G) {
    if (threadIdx.x < 32)
        for (unsigned i = threadIdx.x; i < G; i += 32) {
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst + i));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src + i) : "memory");
        }
}

// block partial of v (all threads) -> dst[blockIdx.x]
__device__ __forceinline__ void cta_partial(double v, double* dst, double* red) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < kWinWarps; ++k) t += red[k];
        dst[blockIdx.x] = t;
    }
}

template <bool DICT, bool LG>
__global__ void __launch_bounds__(kWinBlock, kWinMinBlocks) tau_lanczos_win_kernel(SolveArgs a) {
    __shared__ double smem[kWinWarps + 1];
    __shared__ double red[kWinWarps];
    __shared__ double bc[2];
    extern __shared__ __align__(16) unsigned char dsmem[];
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kWinBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kWinBlock;
    const unsigned epoch0 = *reinterpret_cast<volatile unsigned*>(a.sync.gen);
    Epoch epoch{epoch0, epoch0};
    const WinSmem ws = win_smem_init<0, 24, LG>(dsmem, a);
    float* win = static_cast<float*>(ws.win);
    struct LzRow {
        double isp, w, qp;  // P^-1/2, w_j (unnormalised), q_j-1 of one coordinate
    };
    LzRow* cs = static_cast<LzRow*>(ws.ownT);
    float* uC = static_cast<float*>(a.yC);         // P^-1/2 w_j on C
    float* tR = static_cast<float*>(a.res);        // t' = Theta P^-1/2 w_j on R
    const unsigned G = gridDim.x;
    const uint32_t mw = a.wA.max_win > a.wT.max_win ? a.wA.max_win : a.wT.max_win;
    double* pstage = reinterpret_cast<double*>(static_cast<unsigned char*>(ws.win) + win_align16(mw * 4u));
    double* lz_al = pstage + 2 * G;   // alpha_j
    double* lz_be = lz_al + kLzCap;   // beta_j = |w_j| (beta_0 = |v0 on C|)
    double s2[2] = {0.0, 0.0};
    for (uint64_t i = gthread; i < a.n; i += nthreads) {
        const double v = rng_normal(0x5eedull, i);
        s2[0] += v * v;
    }
    for (uint32_t i = threadIdx.x; i < ws.nrT; i += kWinBlock) {
        const uint32_t c = ws.rT0 + i;
        const double v = rng_normal(0x5eedull, a.C_glob[c]);
        const double isp = a.ispC[c];
        cs[i] = LzRow{isp, v, 0.0};
        uC[c] = static_cast<float>(isp * v);
        s2[1] += v * v;
    }
    grid_sync_reduce<2, kWinBlock>(a.sync, epoch, s2, smem);
    // control state in shared memory (identical in every CTA): keeps the phases' registers
    // for the slice loops
    __shared__ LzCtl ctl;
    if (threadIdx.x == 0) {
        const double beta = sqrt(s2[1]);
        ctl.beta = beta;
        lz_be[0] = beta;
        ctl.r2 = s2[1] / s2[0];
        ctl.lambda = 0.0;
        ctl.check_prev = -1.0;
        ctl.stop_prev = -1;
        ctl.iters = ctl.steps = 0;
        ctl.zero = !(beta > 0.0);
        ctl.breakdown = 0;
        ctl.gap = a.lz_gap;
        ctl.tol = a.lz_tol;
        ctl.done = ctl.zero;
    }
    __syncthreads();
    WinProf pf;
    for (int j = 0; !ctl.done;) {
        // convergence check on T_j (alpha_0..j-1, beta_1..j-1 are known)
        const bool final = ctl.breakdown || j == kLzCap;
        if ((final || (j > 0 && j >= a.lz_first && (j - a.lz_first) % a.lz_every == 0)) &&
            lz_check(lz_al, lz_be, j, final, &ctl))
            break;
        // phase A_j: t' = Theta P^-1/2 w_j and |t'|^2; the partials of |w_j|^2 (phase T_j-1) are
        // staged and summed meanwhile
        double* part = a.sync.part + static_cast<uint64_t>(j & 1) * kRedSlots * G;
        if (j > 0) stage_partials(pstage, a.sync.part + static_cast<uint64_t>((j - 1) & 1) * kRedSlots * G + 3 * G, G);
        pf.side = 0;
        float accA = 0.f;  // a handful of rows per thread: fp32, then fp64 across threads and CTAs
        win_phase<float, float, DICT>(a.wA, ws.uA, ws.usA, ws.nuA, ws.sA, ws.nsA, ws.dA, uC, win,
                                      [&](uint32_t r, double t) {
                                          const float tf = static_cast<float>(t);
                                          tR[r] = tf;
                                          accA = fmaf(tf, tf, accA);
                                      },
                                      pf);
        if (j > 0) {
            const double bb = cta_sum_staged(pstage, G, red);
            if (threadIdx.x == 0) {
                const double beta = sqrt(bb);
                ctl.beta = beta;
                ctl.rb = 1.0 / beta;
                ctl.breakdown = !(beta > 1e-13 * (fabs(lz_al[j - 1]) + lz_be[j - 1]));  // T_j is exact
            }
        } else if (threadIdx.x == 0) {
            ctl.rb = 1.0 / ctl.beta;
        }
        cta_partial(static_cast<double>(accA), part + 2 * G, red);
        grid_sync(a.sync, epoch, smem);
        if (ctl.breakdown) continue;  // (written before the barrier) T_j is exact
        // phase T_j: w_j+1 = M q_j - alpha_j q_j - beta_j q_j-1 on the CTA's coordinates, |w_j+1|^2;
        // alpha_j = |t'|^2 / beta_j^2 from the staged partials of phase A_j
        stage_partials(pstage, part + 2 * G, G);
        pf.side = 3;
        win_phase<float, float, DICT>(
            a.wT, ws.uT, ws.usT, ws.nuT, ws.sT, ws.nsT, ws.dT, tR, win,
            [&](uint32_t c, double g) {
                WBX_ASSERT(c - ws.rT0 < ws.nrT);
                LzRow& st = cs[c - ws.rT0];
                const double rb = ctl.rb;
                const double z = st.isp * g * rb;  // (M q_j)_c
                const double q = st.w * rb;        // q_j
                const double wn = z - ctl.alpha * q - ctl.beta * st.qp;
                st.w = wn;
                st.qp = q;
                uC[c] = static_cast<float>(st.isp * wn);
            },
            pf, [&]() {
                const double S = cta_sum_staged(pstage, G, red);
                if (threadIdx.x == 0) ctl.alpha = S * ctl.rb * ctl.rb;
                __syncthreads();
            });
        if (threadIdx.x == 0) {
            lz_al[j] = ctl.alpha;
            lz_be[j] = ctl.beta;
        }
        __syncthreads();
        double accT = 0.0;
        for (uint32_t i = threadIdx.x; i < ws.nrT; i += kWinBlock) accT = fma(cs[i].w, cs[i].w, accT);
        cta_partial(accT, part + 3 * G, red);
        grid_sync(a.sync, epoch, smem);
        ++j;
    }
    pf.flush();
    if (gthread == 0) {
        const double lambda = ctl.lambda;
        a.out[OUT_TAU] = (ctl.zero || lambda <= 0.0) ? 1.0 : 1.0 / (lambda * a.step_safety);
        a.out[OUT_TAU_ITERS] = ctl.iters;
        a.out[OUT_LAMBDA_MAX] = lambda;
        a.out[OUT_TAU_STEPS] = ctl.steps;
    }
}

// The same Lanczos estimate on the stream engine (fp32 operator stream, fp32 vectors; the
// operators whose windows do not fit: C3, C4 on one GPU). Per coordinate of C: w_j in a.wv,
// q_j-1 in a.uC (fp64, unused by the fp32 power iteration); reductions are not deferred.
__global__ void __launch_bounds__(kBlock, WBX_TAU_MINB) tau_lanczos_kernel(SolveArgs a) {
    __shared__ double smem[kWarpsPerBlock + 1];
    __shared__ double lz_al[kLzCap], lz_be[kLzCap];
    __shared__ LzCtl ctl;
    const int lane = threadIdx.x & 31;
    const uint32_t gwarp = (blockIdx.x * kBlock + threadIdx.x) >> 5;
    const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kBlock;
    const unsigned epoch0 = *reinterpret_cast<volatile unsigned*>(a.sync.gen);
    Epoch epoch{epoch0, epoch0};
    extern __shared__ __align__(16) unsigned char dsmem[];
    Streamer st{};
    st_init(st, dsmem + (threadIdx.x >> 5) * warp_smem_bytes(a.nslots), a.A, a.T, gwarp, nwarps, lane, kLzCap, false,
            a.nslots);
    float* uC = static_cast<float*>(a.yC);  // P^-1/2 w_j on C
    float* tR = static_cast<float*>(a.res); // t' = Theta P^-1/2 w_j on R
    double* qp = a.uC;                      // q_j-1 on C
    double s2[2] = {0.0, 0.0};
    for (uint64_t i = gthread; i < a.n; i += nthreads) {
        const double v = rng_normal(0x5eedull, i);
        s2[0] += v * v;
    }
    for (uint64_t c = gthread; c < a.nC; c += nthreads) {
        const double v = rng_normal(0x5eedull, a.C_glob[c]);
        a.wv[c] = v;
        qp[c] = 0.0;
        uC[c] = static_cast<float>(a.ispC[c] * v);
        s2[1] += v * v;
    }
    grid_sync_reduce<2>(a.sync, epoch, s2, smem);
    if (threadIdx.x == 0) {
        const double beta = sqrt(s2[1]);
        ctl.beta = beta;
        ctl.rb = 1.0 / beta;
        lz_be[0] = beta;
        ctl.r2 = s2[1] / s2[0];
        ctl.lambda = 0.0;
        ctl.check_prev = -1.0;
        ctl.stop_prev = -1;
        ctl.iters = ctl.steps = 0;
        ctl.zero = !(beta > 0.0);
        ctl.done = ctl.zero;
        ctl.breakdown = 0;
        ctl.gap = a.lz_gap;
        ctl.tol = a.lz_tol;
    }
    __syncthreads();
    for (int j = 0; !ctl.done;) {
        const bool final = ctl.breakdown || j == kLzCap;
        if ((final || (j > 0 && j >= a.lz_first && (j - a.lz_first) % a.lz_every == 0)) &&
            lz_check(lz_al, lz_be, j, final, &ctl))
            break;
        // phase A_j: t' = Theta P^-1/2 w_j, |t'|^2 -> alpha_j = |t'|^2 / beta_j^2
        double accA[1] = {0.0};
        st_phase<float, float>(st, a.A, a.T, gwarp, nwarps, lane, st.nA, uC, [](uint32_t) { return 0; },
                               [&](uint32_t r, float t, int) {
                                   tR[r] = t;
                                   accA[0] = fma(static_cast<double>(t), static_cast<double>(t), accA[0]);
                               });
        grid_sync_reduce<1>(a.sync, epoch, accA, smem);
        const double beta = ctl.beta, rb = ctl.rb;
        const double alpha = accA[0] * rb * rb;
        // phase T_j: w_j+1 = M q_j - alpha_j q_j - beta_j q_j-1, |w_j+1|^2 -> beta_j+1
        double accT[1] = {0.0};
        st_phase<float, float>(
            st, a.A, a.T, gwarp, nwarps, lane, st.nT, tR,
            [&](uint32_t c) {
                return c != kNoRow ? make_double3(a.ispC[c], a.wv[c], qp[c]) : make_double3(0.0, 0.0, 0.0);
            },
            [&](uint32_t c, float g, double3 pv) {
                const double z = pv.x * static_cast<double>(g) * rb;  // (M q_j)_c
                const double q = pv.y * rb;                           // q_j
                const double wn = z - alpha * q - beta * pv.z;
                a.wv[c] = wn;
                qp[c] = q;
                uC[c] = static_cast<float>(pv.x * wn);
                accT[0] = fma(wn, wn, accT[0]);
            });
        grid_sync_reduce<1>(a.sync, epoch, accT, smem);
        if (threadIdx.x == 0) {
            lz_al[j] = alpha;
            const double bn = sqrt(accT[0]);
            if (j + 1 < kLzCap) lz_be[j + 1] = bn;
            ctl.beta = bn;
            ctl.rb = 1.0 / bn;
            ctl.breakdown = !(bn > 1e-13 * (fabs(alpha) + beta));  // T_j+1 is exact
        }
        __syncthreads();
        ++j;
    }
    st_drain(st);
    if (gthread == 0) {
        const double lambda = ctl.lambda;
        a.out[OUT_TAU] = (ctl.zero || lambda <= 0.0) ? 1.0 : 1.0 / (lambda * a.step_safety);
        a.out[OUT_TAU_ITERS] = ctl.iters;
        a.out[OUT_LAMBDA_MAX] = lambda;
        a.out[OUT_TAU_STEPS] = ctl.steps;
    }
}

// ---------------------------------------------------------------- batched FISTA (C5)
// B independent images sharing Theta_K, P, w, lambda and tau (BASELINE config C5): the
// operator stream is read once per B right-hand sides (SpMM). Vectors are interleaved
// [coordinate][B] so a gathered column is one 4*B-byte segment (B=8: one 32-B sector).
template <int B, typename Pre, typename Post>
__device__ __forceinline__ void st_phase_batch(Streamer& st, const SellView& A, const SellView& T, uint32_t gwarp,
                                               uint32_t nwarps, int lane, uint32_t count,
                                               const float* __restrict__ x, Pre pre, Post post) {
    static_assert(B % 4 == 0, "batch must be a multiple of 4");
    constexpr int V = B / 4;
    for (uint32_t i = 0; i < count; ++i) {
        const uint64_t e = st.consumed;
        const unsigned slot = static_cast<unsigned>(e % st.ns);
        mbar_wait(st.bars + slot, static_cast<unsigned>((e / st.ns) & 1u));
        const uint32_t meta = st.meta[slot];
        const int np = static_cast<int>(meta & 0xffu);
        const uint4* rec = st.slots + slot * kRecU4;
        const uint32_t info = reinterpret_cast<const uint32_t*>(rec)[lane];
        const auto pv = pre(info == kNoRow ? kNoRow : (info & kRowMask));
        const uint4* p = rec + 8 + lane;
        float acc[B];
#pragma unroll
        for (int b = 0; b < B; ++b) acc[b] = 0.f;
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // two halves of 4 element pairs each
            uint4 q[4];
            float4 g[8][V];
#pragma unroll
            for (int j = 0; j < 4; ++j) q[j] = (4 * h + j) < np ? p[(4 * h + j) * kWarp] : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const bool on = (4 * h + j) < np;
                    g[2 * j][v] = on ? reinterpret_cast<const float4*>(x + static_cast<uint64_t>(q[j].y) * B)[v]
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                    g[2 * j + 1][v] = on ? reinterpret_cast<const float4*>(x + static_cast<uint64_t>(q[j].w) * B)[v]
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float v0 = __uint_as_float(q[j].x), v1 = __uint_as_float(q[j].z);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    acc[4 * v + 0] = fmaf(v0, g[2 * j][v].x, acc[4 * v + 0]);
                    acc[4 * v + 1] = fmaf(v0, g[2 * j][v].y, acc[4 * v + 1]);
                    acc[4 * v + 2] = fmaf(v0, g[2 * j][v].z, acc[4 * v + 2]);
                    acc[4 * v + 3] = fmaf(v0, g[2 * j][v].w, acc[4 * v + 3]);
                    acc[4 * v + 0] = fmaf(v1, g[2 * j + 1][v].x, acc[4 * v + 0]);
                    acc[4 * v + 1] = fmaf(v1, g[2 * j + 1][v].y, acc[4 * v + 1]);
                    acc[4 * v + 2] = fmaf(v1, g[2 * j + 1][v].z, acc[4 * v + 2]);
                    acc[4 * v + 3] = fmaf(v1, g[2 * j + 1][v].w, acc[4 * v + 3]);
                }
            }
        }
        // segment partials -> head lane, fixed order (as combine_info, B values)
        const uint32_t m = meta >> 8;
        const uint32_t nseg = info == kNoRow ? 1u : (info >> 27);
        const uint32_t maxseg = __reduce_max_sync(0xffffffffu, nseg);
        for (uint32_t j = 1; j < maxseg; ++j) {
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const float t = __shfl_down_sync(0xffffffffu, acc[b], j * m);
                if (j < nseg) acc[b] += t;
            }
        }
        __syncwarp();
        st.consumed = e + 1;
        if (st.issued < st.limit) st_issue(st, A, T, gwarp, nwarps, lane);
        if (info != kNoRow) post(info & kRowMask, acc, pv);
    }
}

template <int B>
__global__ void __launch_bounds__(kBlock, WBX_FISTA_MINB) fista_batch_kernel(SolveArgs a) {
    __shared__ double smem[kWarpsPerBlock + 1];
    const int lane = threadIdx.x & 31;
    const uint32_t gwarp = (blockIdx.x * kBlock + threadIdx.x) >> 5;
    const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kBlock;
    const unsigned epoch0 = *reinterpret_cast<volatile unsigned*>(a.sync.gen);
    Epoch epoch{epoch0, epoch0};
    float* yC = static_cast<float*>(a.yC);   // [nC][B]
    float* xpC = static_cast<float*>(a.xpC);  // [nC][B]
    float* res = static_cast<float*>(a.res);  // [nR][B]
    float* x0R = static_cast<float*>(a.x0R);  // [nR][B]
    float* tpC = static_cast<float*>(a.tpC);  // [nC]
    float* thrC = static_cast<float*>(a.thrC);
    const double tau = a.out[OUT_TAU];
    extern __shared__ __align__(16) unsigned char dsmem[];
    Streamer st{};
    st_init(st, dsmem + (threadIdx.x >> 5) * warp_smem_bytes(a.nslots), a.A, a.T, gwarp, nwarps, lane,
            static_cast<uint64_t>(a.max_iters), false, a.nslots);
    const uint64_t n = a.n;
    for (uint64_t c = gthread; c < a.nC; c += nthreads) {
        const uint32_t g = a.C_glob[c];
        for (int b = 0; b < B; ++b) {
            const float v = static_cast<float>(a.x0_full[b * n + g]);
            yC[c * B + b] = v;
            xpC[c * B + b] = v;
        }
        tpC[c] = static_cast<float>(tau / a.pC[c]);
        thrC[c] = static_cast<float>(thr_exact(tau, a.lambda, a.wC[c], a.pC[c]));
    }
    for (uint64_t r = gthread; r < a.nR; r += nthreads) {
        const uint32_t g = a.R_glob[r];
        for (int b = 0; b < B; ++b) x0R[r * B + b] = static_cast<float>(a.x0_full[b * n + g]);
    }
    for (int b = 0; b < B; ++b) {
        SolveArgs ab = a;
        ab.x0_full = a.x0_full + b * n;
        ab.x_full = a.x_full + b * n;
        decoupled_pass<float>(ab, tau, a.max_iters, 0, gthread, nthreads, nullptr, nullptr, 0);
    }
    grid_sync(a.sync, epoch, smem);
    struct VecB {
        float v[B];
    };
    for (int k = 1; k <= a.max_iters; ++k) {
        st_phase_batch<B>(
            st, a.A, a.T, gwarp, nwarps, lane, st.nA, yC,
            [&](uint32_t r) {
                VecB q;
#pragma unroll
                for (int b = 0; b < B; ++b) q.v[b] = r != kNoRow ? x0R[static_cast<uint64_t>(r) * B + b] : 0.f;
                return q;
            },
            [&](uint32_t r, const float (&acc)[B], const VecB& x0) {
#pragma unroll
                for (int b = 0; b < B; ++b) res[static_cast<uint64_t>(r) * B + b] = acc[b] - x0.v[b];
            });
        grid_sync(a.sync, epoch, smem);
        const float beta = a.beta32[k - 1];
        struct CoordB {
            float y[B], xp[B], tp, thr;
        };
        st_phase_batch<B>(
            st, a.A, a.T, gwarp, nwarps, lane, st.nT, res,
            [&](uint32_t c) {
                CoordB q;
                const bool on = c != kNoRow;
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    q.y[b] = on ? yC[static_cast<uint64_t>(c) * B + b] : 0.f;
                    q.xp[b] = on ? xpC[static_cast<uint64_t>(c) * B + b] : 0.f;
                }
                q.tp = on ? tpC[c] : 0.f;
                q.thr = on ? thrC[c] : 0.f;
                return q;
            },
            [&](uint32_t c, const float (&g)[B], const CoordB& q) {
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const float z0 = fmaf(-q.tp, g[b], q.y[b]);
                    const float xn = Prec<float>::prox(z0, q.thr);
                    yC[static_cast<uint64_t>(c) * B + b] = fmaf(beta, xn - q.xp[b], xn);
                    xpC[static_cast<uint64_t>(c) * B + b] = xn;
                }
            });
        grid_sync(a.sync, epoch, smem);
    }
    st_drain(st);
    if (gthread == 0) a.out[OUT_ITERS_USED] = a.max_iters;
    for (uint64_t c = gthread; c < a.nC; c += nthreads) {
        const uint32_t g = a.C_glob[c];
        for (int b = 0; b < B; ++b) a.x_full[b * n + g] = static_cast<double>(xpC[c * B + b]);
    }
}

#include "stencil_kernel.cuh"

// Decoupled pass as its own kernel (tracking mode: per-iteration sums, then the final
// write with the iteration count the solve actually used).
template <typename T>
__global__ void __launch_bounds__(kBlock) decoupled_kernel(SolveArgs a, int mode, double* wreg, double* wsup,
                                                           const double* out) {
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kBlock;
    const double tau = out[OUT_TAU];
    const int K = mode == 0 ? static_cast<int>(out[OUT_ITERS_USED]) : a.max_iters;
    decoupled_pass<T>(a, tau, K, mode, gthread, nthreads, wreg, wsup, nthreads / 32);
}

// wreg/wsup [K][nwarps] -> dec_reg/dec_supp [K]: one warp per k, lane-strided partial sums
// folded by a fixed shuffle tree (deterministic)
__global__ void reduce_rows_kernel(const double* w, uint64_t nwarps, int K, double* outp) {
    const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (k >= K) return;
    double s = 0.0;
    for (uint64_t j = lane; j < nwarps; j += 32) s += w[static_cast<uint64_t>(k) * nwarps + j];
    s = warp_sum(s);
    if (lane == 0) outp[k] = s;
}

__global__ void set_tau_kernel(double* out, double tau) {
    out[OUT_TAU] = tau;
    out[OUT_TAU_ITERS] = 0;
    out[OUT_TAU_STEPS] = 0;
}

__global__ void clamp_kernel(double* u, uint64_t n) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) u[i] = fmin(fmax(u[i], 0.0), 1.0);  // std::clamp(v, 0, 1), waveblur.cpp:297
}

}  // namespace
}  // namespace wbx

// ---------------------------------------------------------------- solver object
struct wbx_solver {
    wbx_ctx* ctx = nullptr;
    const wbx_op* op = nullptr;
    wbx_basis* basis = nullptr;
    uint64_t n = 0;
    double lambda = 0.0;
    wbx_solver_cfg cfg{};
    int accelerate = 1;
    int batch = 1;  // images per solve (C5): 1, 4 or 8
    wbx::DevBuf<double> pC, wC, ispC, w_full, p_full, beta64;
    wbx::DevBuf<float> beta32;
    wbx::DevBuf<unsigned char> state;  // yC, xpC, res, x0R, tpC, thrC (T-typed)
    wbx::DevBuf<double> wv, uC, t64, out, energies, dec_reg, dec_supp, wreg, wsup, part, red;
    wbx::DevBuf<unsigned long long> supports;
    wbx::DevBuf<unsigned> gen, arrive;
    wbx::DevBuf<unsigned long long> trace;  // WBX_TRACE_FILE diagnostics
    uint64_t trace_cap = 0;
    wbx::DevBuf<double> u0, x0full, xfull, uout;
    int grid_fista = 0, grid_tau = 0;
    int nslots = 3;  // TMA slots in flight per warp
    // window engine (fp32 single-image solves whose per-CTA windows fit shared memory)
    bool win = false, win_dict = false, tau_win64 = false, tau_lanczos = false;
    bool win_track = false;  // tracked solves (energies / supports / ref_energy) on the window engine
    bool win_lists_global = false;  // window index lists in global memory (large windows)
    bool tau_stream_lz = false;     // window FISTA with the streamed engine's Lanczos step estimate
    unsigned win_smem_track = 0;
    int grid_tau_lz = 0;
    int grid_win = 0;
    unsigned win_smem_fista = 0, win_smem_tau = 0;
    std::shared_ptr<wbx::WinPair> wp;  // window layouts (owned by the operator's cache)
    // stencil engine (stationary operators with their generator groups attached)
    bool stencil = false;
    int grid_st = 0;
    unsigned st_smem = 0;
    std::shared_ptr<wbx::StencilPlan> sp;  // owned by the operator's cache
    // block-Fourier step estimate (circ_tau.cu) for translation-invariant operators
    bool tau_circ = false;
    bool fista_circ = false;  // spectral FISTA engine (circ_fista_kernel): fp64, untracked single images
    std::shared_ptr<wbx::CircPlan> circ;  // owned by the operator's cache
    wbx::DevBuf<double> circ_isp, circ_work;
    wbx::DevBuf<double2> circ_gram, circ_T;
    wbx::DevBuf<double> circ_track;  // tracked spectral solves: per-CTA / per-warp energy partials
    wbx::DevBuf<unsigned> circ_counter;
    wbx::DevBuf<double> bwork;  // batches: the DWT work buffers of every image (2 n per image)
    uint32_t circ_slots = 1;  // batch images per spectral launch (circ_fista_slots)
    wbx::DevBuf<float> yF, resF;
    int dec_grid = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_mid = nullptr, ev_it0 = nullptr, ev_in = nullptr;
    cudaStream_t copy_stream = nullptr;  // host->device image copies overlapping the step estimate
    bool input_pending = false;          // ev_in marks a pending copy of the input image
    uint64_t last_launches = 0;
    float last_solve_ms = 0.f;
    // CUDA graphs of the deblur (WBX_GRAPH=0 disables): the step estimate, and analyze +
    // iterations + synthesize (+ clamp) for the last (u0, u, clamp) pointers
    cudaGraphExec_t g_tau = nullptr, g_rest = nullptr, g_an = nullptr;  // g_an: analyze (side stream)
    cudaEvent_t ev_an = nullptr;  // the analysis of the input is done (side stream -> main stream)
    cudaStream_t aux_stream = nullptr;  // fork / join inside the step estimate (G_f beside v0's transform)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    const double* g_an_u0 = nullptr;
    uint64_t g_an_launches = 0;
    double* g_u = nullptr;
    int g_clamp = -1;
    uint64_t g_tau_launches = 0, g_rest_launches = 0;
    bool graphs_off = false;
};

namespace wbx {

namespace {

// dynamic shared memory of the persistent kernels: the per-warp TMA slot rings (fp32)
template <typename T>
unsigned dyn_smem(int nslots) {
    return sizeof(T) == 4 ? kWarpsPerBlock * warp_smem_bytes(nslots) : 0u;
}

int blocks_per_sm(const void* kernel, unsigned smem) {
    if (smem > 0)
        WBX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    WBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, smem));
    if (per_sm < 1) fail(WBX_CUDA_ERROR, "solver kernel cannot be resident");
    // tuning override: WBX_SOLVER_BLOCKS_PER_SM (clamped to what is co-resident)
    if (const char* e = std::getenv("WBX_SOLVER_BLOCKS_PER_SM")) {
        const int want = std::atoi(e);
        if (want >= 1 && want < per_sm) per_sm = want;
    }
    return per_sm;
}

int env_int(const char* name, int dflt, int lo, int hi) {
    const char* e = std::getenv(name);
    return e ? std::max(lo, std::min(hi, std::atoi(e))) : dflt;
}

template <typename T>
SolveArgs make_args(wbx_solver* s, const double* x0_full, double* x_full) {
    const wbx_op* op = s->op;
    SolveArgs a{};
    a.A = view_of(op->A);
    a.T = view_of(op->T);
    a.R_glob = op->R_glob.p;
    a.C_glob = op->C_glob.p;
    a.isC = op->isC.p;
    a.isR = op->isR.p;
    a.nR = static_cast<uint32_t>(op->nR);
    a.nC = static_cast<uint32_t>(op->nC);
    a.n = op->n;
    a.x0_full = x0_full;
    a.x_full = x_full;
    a.w_full = s->w_full.p;
    a.p_full = s->p_full.p;
    a.pC = s->pC.p;
    a.wC = s->wC.p;
    a.ispC = s->ispC.p;
    a.beta64 = s->beta64.p;
    a.beta32 = s->beta32.p;
    a.lambda = s->lambda;
    a.tau_given = s->cfg.tau;
    a.tau_from_device = 1;
    a.step_safety = s->cfg.step_safety;
    a.ref_energy = s->cfg.ref_energy;
    a.rel_tol = s->cfg.rel_energy_tol;
    a.max_iters = static_cast<int>(s->cfg.max_iters);
    a.stop_on_ref = std::isfinite(s->cfg.ref_energy) ? 1 : 0;
    a.track = (s->cfg.track_energy || s->cfg.track_support || a.stop_on_ref) ? 1 : 0;
    a.decoupled_inline = a.track ? 0 : 1;
    const uint64_t nC = op->nC, nR = op->nR;
    unsigned char* st = s->state.p;
    auto carve = [&](uint64_t count) {
        void* p = st;
        st += ((count * sizeof(T) + 255) / 256) * 256;
        return p;
    };
    const uint64_t B = static_cast<uint64_t>(s->batch);
    a.yC = carve(nC * B);
    a.xpC = carve(nC * B);
    a.res = carve(nR * B);
    a.x0R = carve(nR * B);
    a.tpC = carve(nC);
    a.thrC = carve(nC);
    a.wv = s->wv.p;
    a.uC = s->uC.p;
    a.t64 = s->t64.p;
    a.dec_reg = s->dec_reg.p;
    a.dec_supp = s->dec_supp.p;
    a.out = s->out.p;
    a.energies = s->energies.p;
    a.supports = s->supports.p;
    a.sync.gen = s->gen.p;
    a.sync.arrive = s->arrive.p;
    a.sync.part = s->part.p;
    a.sync.red = s->red.p;
    a.sync.trace = s->trace.p;
    a.sync.trace_cap = static_cast<unsigned>(s->trace_cap);
    a.nslots = s->nslots;
    a.lz_first = env_int("WBX_LZ_FIRST", 48, 1, kLzCap);
    a.lz_every = env_int("WBX_LZ_EVERY", 4, 1, kLzCap);
    a.lz_gap = env_int("WBX_LZ_GAP", 4, 1, kLzCap);
    a.lz_tol = std::getenv("WBX_LZ_TOL") ? std::atof(std::getenv("WBX_LZ_TOL")) : 1e-8;
    if (s->win) {
        a.wA = view_of(s->wp->A);
        a.wT = view_of(s->wp->T);
        a.win_lists_global = s->win_lists_global ? 1 : 0;
    }
    if (s->stencil) {
        a.st = view_of(*s->sp);
        a.st_fill = env_int("WBX_ST_FILL", 0, 0, 2);
        a.yF = s->yF.p;
        a.resF = s->resF.p;
    }
    {
        const char* e = std::getenv("WBX_BARRIER");
        a.sync.mode = !e ? 2 : std::string(e) == "allpoll" ? 1 : std::string(e) == "master" ? 0 : 2;
        a.sync.groups = env_int("WBX_BARRIER_GROUPS", 1, 1, kMaxCounterGroups);
    }
    return a;
}

template <bool LG>
const void* tau_win_fn_lg(bool dict, bool w64, bool lanczos) {
    if (lanczos)
        return dict ? reinterpret_cast<const void*>(tau_lanczos_win_kernel<true, LG>)
                    : reinterpret_cast<const void*>(tau_lanczos_win_kernel<false, LG>);
    if (dict)
        return w64 ? reinterpret_cast<const void*>(tau_win_kernel<true, double, LG>)
                   : reinterpret_cast<const void*>(tau_win_kernel<true, float, LG>);
    return w64 ? reinterpret_cast<const void*>(tau_win_kernel<false, double, LG>)
               : reinterpret_cast<const void*>(tau_win_kernel<false, float, LG>);
}

// the window kernels by value format (dictionary / full) and index-list placement (smem / global)
const void* tau_win_fn(bool dict, bool w64, bool lanczos, bool lg) {
    return lg ? tau_win_fn_lg<true>(dict, w64, lanczos) : tau_win_fn_lg<false>(dict, w64, lanczos);
}

const void* fista_win_fn(bool dict, bool lg) {
    if (dict)
        return lg ? reinterpret_cast<const void*>(fista_win_kernel<true, true>)
                  : reinterpret_cast<const void*>(fista_win_kernel<true, false>);
    return lg ? reinterpret_cast<const void*>(fista_win_kernel<false, true>)
              : reinterpret_cast<const void*>(fista_win_kernel<false, false>);
}

const void* track_win_fn(bool dict, bool lg) {
    if (dict)
        return lg ? reinterpret_cast<const void*>(fista_win_track_kernel<true, true>)
                  : reinterpret_cast<const void*>(fista_win_track_kernel<true, false>);
    return lg ? reinterpret_cast<const void*>(fista_win_track_kernel<false, true>)
              : reinterpret_cast<const void*>(fista_win_track_kernel<false, false>);
}

void launch_coop_smem(const void* kernel, int grid, unsigned smem, SolveArgs& a, cudaStream_t st,
                      int block = kBlock) {
    if (a.sync.mode == 2)  // the counter barrier counts from zero in every launch
        WBX_CUDA(cudaMemsetAsync(a.sync.gen + kCounterWord, 0, 32u * kMaxCounterGroups * sizeof(unsigned), st));
    void* params[] = {&a};
    WBX_CUDA(cudaLaunchCooperativeKernel(kernel, dim3(grid), dim3(block), params, smem, st));
}

template <typename T>
void launch_coop(const void* kernel, int grid, SolveArgs& a, cudaStream_t st) {
    launch_coop_smem(kernel, grid, dyn_smem<T>(a.nslots), a, st);
}

template <typename T>
void run_tau(wbx_solver* s, const double* x0_full, double* x_full, cudaStream_t st) {
    SolveArgs a = make_args<T>(s, x0_full, x_full);
    wbx_ctx* ctx = s->ctx;
    WBX_CUDA(cudaMemsetAsync(s->out.p, 0, s->out.bytes(), st));
    // step: estimate_step on the device, or the given one
    if (s->cfg.tau > 0.0) {
        set_tau_kernel<<<1, 1, 0, st>>>(s->out.p, s->cfg.tau);
    } else if (s->tau_circ) {  // translation-invariant operator: block-Fourier power iteration
        circ_tau_launch(ctx, *s->circ, s->circ_isp.p, s->cfg.step_safety, s->circ_work.p, s->circ_gram.p, s->out.p,
                        st, s->aux_stream, s->ev_fork, s->ev_join);
        return;
    } else if (s->win && !s->tau_stream_lz) {
        const void* k = tau_win_fn(s->win_dict, s->tau_win64, s->tau_lanczos, s->win_lists_global);
        launch_coop_smem(k, s->grid_win, s->win_smem_tau, a, st, kWinBlock);
    } else if (sizeof(T) == 4 && (s->tau_lanczos || s->tau_stream_lz)) {
        launch_coop<T>(reinterpret_cast<const void*>(tau_lanczos_kernel), s->grid_tau_lz, a, st);
    } else {
        launch_coop<T>(reinterpret_cast<const void*>(tau_kernel<T>), s->grid_tau, a, st);
    }
    count_launch(ctx);
    WBX_CUDA(cudaGetLastError());
}

// the iteration kernel(s) after run_tau (tau on the device in out[OUT_TAU])
template <typename T>
void run_iters(wbx_solver* s, const double* x0_full, double* x_full, cudaStream_t st) {
    SolveArgs a = make_args<T>(s, x0_full, x_full);
    wbx_ctx* ctx = s->ctx;
    if (s->fista_circ && !a.stop_on_ref) {  // spectral engine (translation-invariant operator)
        if (!s->tau_circ || s->cfg.tau > 0.0) circ_gram_launch(ctx, *s->circ, s->circ_gram.p, st);
        CircProblem pr{a.x0_full, a.w_full, a.p_full, a.x_full, a.isC, a.beta64, a.lambda, a.max_iters, a.out};
        if (a.track) {  // energies / supports of every iterate (solver.cpp:130-137)
            pr.track_work = s->circ_track.p;
            pr.energies = s->energies.p;
            pr.supports = s->supports.p;
        }
        // a batch (C5): circ_slots images per launch, images back to back in x0_full / x_full
        const uint32_t B = static_cast<uint32_t>(s->batch);
        for (uint32_t b0 = 0; b0 < B; b0 += s->circ_slots) {
            pr.nimg = std::min(s->circ_slots, B - b0);
            pr.x0_full = x0_full + static_cast<uint64_t>(b0) * s->n;
            pr.x_full = x_full + static_cast<uint64_t>(b0) * s->n;
            circ_fista_launch(ctx, *s->circ, pr, s->circ_gram.p, s->circ_T.p, s->circ_counter.p, st);
        }
        return;
    }
    if (s->stencil && !a.track && s->batch == 1) {
        a.isC = a.st.coupled;  // the decoupled pass: coordinates outside the Theta^T output bands
        launch_coop_smem(reinterpret_cast<const void*>(fista_stencil_kernel), s->grid_st, s->st_smem, a, st, kStBlock);
        count_launch(ctx);
        WBX_CUDA(cudaGetLastError());
        return;
    }
    const bool win = s->win && !a.track && s->batch == 1;
    if (win) {
        const void* k = fista_win_fn(s->win_dict, s->win_lists_global);
        launch_coop_smem(k, s->grid_win, s->win_smem_fista, a, st, kWinBlock);
        count_launch(ctx);
        WBX_CUDA(cudaGetLastError());
        return;
    }
    if (s->batch > 1) {  // C5: B images per solve (fp32, no tracking; checked at creation)
        const void* k = s->batch == 4 ? reinterpret_cast<const void*>(fista_batch_kernel<4>)
                                      : reinterpret_cast<const void*>(fista_batch_kernel<8>);
        launch_coop<T>(k, s->grid_fista, a, st);
        count_launch(ctx);
        WBX_CUDA(cudaGetLastError());
        return;
    }
    if (!a.track) {
        launch_coop<T>(reinterpret_cast<const void*>(fista_kernel<T>), s->grid_fista, a, st);
        count_launch(ctx);
        WBX_CUDA(cudaGetLastError());
        return;
    }
    // Tracking (energies / supports / ref_energy stopping rule, solver.cpp:130-150):
    // decoupled per-iteration sums with the tau on device, reduced; tracked solve;
    // decoupled final write at the iteration count used.
    const uint64_t nthreads = static_cast<uint64_t>(s->dec_grid) * kBlock;
    const uint64_t nwarps = nthreads / 32;
    const int K = a.max_iters;
    if (K > 0) {
        WBX_CUDA(cudaMemsetAsync(s->wreg.p, 0, s->wreg.bytes(), st));
        WBX_CUDA(cudaMemsetAsync(s->wsup.p, 0, s->wsup.bytes(), st));
        // without the ref_energy rule the iteration count is known: one pass also writes x_K
        decoupled_kernel<T><<<s->dec_grid, kBlock, 0, st>>>(a, a.stop_on_ref ? 1 : 2, s->wreg.p, s->wsup.p, s->out.p);
        reduce_rows_kernel<<<(K * 32 + 255) / 256, 256, 0, st>>>(s->wreg.p, nwarps, K, s->dec_reg.p);
        reduce_rows_kernel<<<(K * 32 + 255) / 256, 256, 0, st>>>(s->wsup.p, nwarps, K, s->dec_supp.p);
        count_launch(ctx, 3);
    }
    if (s->win_track) {  // the window engine with energy / support tracking
        const void* k = track_win_fn(s->win_dict, s->win_lists_global);
        launch_coop_smem(k, s->grid_win, s->win_smem_track, a, st, kWinBlock);
    } else {
        launch_coop<T>(reinterpret_cast<const void*>(fista_kernel<T>), s->grid_fista, a, st);
    }
    count_launch(ctx);
    if (a.stop_on_ref || K == 0) {  // x_K of the decoupled coordinates at the count actually used
        decoupled_kernel<T><<<s->dec_grid, kBlock, 0, st>>>(a, 0, nullptr, nullptr, s->out.p);
        count_launch(ctx);
    }
    WBX_CUDA(cudaGetLastError());
}

// The operator's block-Fourier step-estimate plan for the basis's layout (cached on the operator)
// (the solver's basis, or the layout attached to the operator: the drop-in fista() has no basis)
std::shared_ptr<CircPlan> circ_plan_for(const wbx_op* op, const wbx_basis* basis) {
    std::lock_guard<std::mutex> g(op->win_mu);
    const uint32_t ndim = basis ? basis->ndim : op->l_ndim, J = basis ? basis->J : op->l_J;
    const uint64_t* dims = basis ? basis->dims : op->l_dims;
    const std::vector<wbx_band>& bands = basis ? basis->bands : op->l_bands;
    std::vector<uint64_t> key{ndim, dims[0], ndim == 2 ? dims[1] : 1, J};
    auto it = op->circ_cache.find(key);
    if (it != op->circ_cache.end()) return it->second;
    auto p = circ_analyze(op, ndim, dims, J, bands);
    op->circ_cache[key] = p;
    return p;
}

// The operator's window layouts for grid size G, built on first use and cached on the operator
std::shared_ptr<WinPair> win_layout(const wbx_op* op, uint32_t G, cudaStream_t st) {
    std::lock_guard<std::mutex> g(op->win_mu);
    auto it = op->win_cache.find(G);
    if (it != op->win_cache.end()) return it->second;
    auto p = std::make_shared<WinPair>();
    try {
        // window placement: chunk layout (16-byte fills, chunks in source order; default, or
        // bank-aware chunk slots with WBX_WIN_PLACE=chunk-bank), or per-entry slots, bank-aware
        // (=bank, round 1's default) or in source order (=sorted)
        const char* pl = std::getenv("WBX_WIN_PLACE");
        const bool chunk = !pl || std::string(pl).rfind("chunk", 0) == 0;
        build_win(p->A, op->hA, G, st, 'A', chunk);
        build_win(p->T, op->hT, G, st, 'T', chunk);
        p->A.src_len = static_cast<uint32_t>(op->nC);  // A rows gather C-space vectors
        p->T.src_len = static_cast<uint32_t>(op->nR);
        WBX_CUDA(cudaStreamSynchronize(st));  // usable from any stream of the device
        p->ok = true;
    } catch (const Error& e) {
        if (e.status != WBX_TOO_LARGE) throw;
        p = std::make_shared<WinPair>();  // not representable at this G (ok == false)
    }
    op->win_cache[G] = p;
    return p;
}

template <typename T>
void alloc_state(wbx_solver* s) {
    const wbx_op* op = s->op;
    auto rnd = [](uint64_t count) { return ((count * sizeof(T) + 255) / 256) * 256; };
    const uint64_t B = static_cast<uint64_t>(s->batch);
    s->state.alloc(2 * rnd(op->nC * B) + 2 * rnd(op->nC) + 2 * rnd(op->nR * B) + 256);
    s->nslots = 3;
    if (const char* e = std::getenv("WBX_SLOTS")) s->nslots = std::max(1, std::min(kMaxSlots, std::atoi(e)));
    s->grid_fista = blocks_per_sm(reinterpret_cast<const void*>(fista_kernel<T>), dyn_smem<T>(s->nslots)) * s->ctx->num_sms;
    s->grid_tau = blocks_per_sm(reinterpret_cast<const void*>(tau_kernel<T>), dyn_smem<T>(s->nslots)) * s->ctx->num_sms;
    // Lanczos tau on the stream engine (fp32; overridden below when the window engine runs)
    s->tau_lanczos = sizeof(T) == 4 && !(std::getenv("WBX_TAU") && std::string(std::getenv("WBX_TAU")) == "power");
    if (sizeof(T) == 4)
        s->grid_tau_lz =
            blocks_per_sm(reinterpret_cast<const void*>(tau_lanczos_kernel), dyn_smem<T>(s->nslots)) * s->ctx->num_sms;
    if (s->batch == 4)
        s->grid_fista = blocks_per_sm(reinterpret_cast<const void*>(fista_batch_kernel<4>), dyn_smem<T>(s->nslots)) * s->ctx->num_sms;
    else if (s->batch == 8)
        s->grid_fista = blocks_per_sm(reinterpret_cast<const void*>(fista_batch_kernel<8>), dyn_smem<T>(s->nslots)) * s->ctx->num_sms;
    // window engine: fp32 (single images; batches use it for tau); try 2 then 1 CTA per SM;
    // fall back to the streamed engine if a CTA's window does not fit (WBX_ENGINE=stream
    // forces the fallback)
    const char* eng = std::getenv("WBX_ENGINE");
    if (sizeof(T) == 4 && !(eng && std::string(eng) == "stream")) {  // batches use it for tau
        // index lists in shared memory first; for windows too large for both lists and window,
        // the lists in global memory (read by the fills) before giving up CTAs per SM
        for (int attempt = 0; attempt < 2 * kWinMinBlocks && !s->win; ++attempt) {
            const int bps = kWinMinBlocks - attempt / 2;
            const bool lg = (attempt & 1) != 0;
            if (const char* wl = std::getenv("WBX_WIN_LISTS")) {  // diagnostics: force one placement
                if ((std::string(wl) == "smem" && lg) || (std::string(wl) == "global" && !lg)) continue;
            }
            const uint32_t G = static_cast<uint32_t>(bps * s->ctx->num_sms);
            s->wp = win_layout(s->op, G, s->ctx->stream);
            if (!s->wp->ok) continue;  // a window exceeded 16-bit local indices
            const WinView vA = view_of(s->wp->A), vT = view_of(s->wp->T);
            const unsigned mu = std::max(s->wp->A.max_win, s->wp->T.max_win);
            s->win_smem_fista = win_smem_head<4, 16>(vA, vT, lg) + mu * 4u;
            // fp64 windows (diagnostics) need per-entry window layouts (WBX_WIN_PLACE=bank)
            s->tau_win64 = std::getenv("WBX_TAU_WINDOW") && std::string(std::getenv("WBX_TAU_WINDOW")) == "64" &&
                           !s->wp->A.chunk;
            // tau by Lanczos + the power iteration on the tridiagonal (tau_lanczos_win_kernel);
            // WBX_TAU=power runs the literal power iteration
            // (falls back to the power iteration when its state does not fit next to the window)
            const unsigned limit = bps == 1 ? 220u * 1024u : (227u * 1024u) / bps - 2048u;
            s->tau_lanczos = !s->tau_win64 && !(std::getenv("WBX_TAU") && std::string(std::getenv("WBX_TAU")) == "power");
            const unsigned smem_lz = win_smem_head<0, 24>(vA, vT, lg) + win_align16(mu * 4u) + 16u * G +  // + partials
                                     16u * kLzCap;                                                     // + alpha, beta
            // the Lanczos state does not fit next to the window: the streamed engine's Lanczos
            // estimate (60-odd steps) rather than the window power iteration (200)
            s->tau_stream_lz = s->tau_lanczos && smem_lz > limit;
            if (s->tau_lanczos && smem_lz > limit) s->tau_lanczos = false;
            s->win_smem_tau = s->tau_lanczos ? smem_lz
                                             : win_smem_head<0, 16>(vA, vT, lg) + win_align16(mu * (s->tau_win64 ? 8u : 4u)) +
                                                   16u * G;  // + partials staging
            s->win_dict = vA.max_dict > 0 && vT.max_dict > 0;
            const void* kf = fista_win_fn(s->win_dict, lg);
            const void* kt = tau_win_fn(s->win_dict, s->tau_win64, s->tau_lanczos, lg);
            if (std::getenv("WBX_VERBOSE"))
                std::fprintf(stderr, "wbx window engine: try G=%u lists %s smem fista/tau=%u/%u limit %u\n", G,
                             lg ? "global" : "smem", s->win_smem_fista, s->win_smem_tau, limit);
            if (std::max(s->win_smem_fista, s->win_smem_tau) > limit) continue;
            WBX_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(s->win_smem_fista)));
            WBX_CUDA(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(s->win_smem_tau)));
            int pf = 0, pt = 0;
            WBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pf, kf, kWinBlock, s->win_smem_fista));
            WBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pt, kt, kWinBlock, s->win_smem_tau));
            if (std::getenv("WBX_VERBOSE"))
                std::fprintf(stderr, "wbx window engine: G=%u occupancy fista/tau=%d/%d\n", G, pf, pt);
            if (pf < bps || pt < bps) continue;
            s->grid_win = static_cast<int>(G);
            s->win = true;
            s->win_lists_global = lg;
            // the tracked variant keeps Theta x_k-1 next to x0 per own row (+4 B per row)
            s->win_smem_track = win_smem_head<8, 16>(vA, vT, lg) + mu * 4u;
            if (s->win_smem_track <= limit && !(std::getenv("WBX_TRACK_ENGINE") &&
                                                std::string(std::getenv("WBX_TRACK_ENGINE")) == "stream")) {
                const void* kk = track_win_fn(s->win_dict, lg);
                WBX_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(s->win_smem_track)));
                int pk = 0;
                WBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pk, kk, kWinBlock, s->win_smem_track));
                s->win_track = pk >= bps;
            }
            if (std::getenv("WBX_VERBOSE"))
                std::fprintf(stderr,
                             "wbx window engine: G=%u max_u A/T=%u/%u max_rows A/T=%u/%u max_slices A/T=%u/%u "
                             "dict floats A/T=%u/%u rec bytes A/T=%llu/%llu smem fista/tau=%u/%u\n",
                             G, s->wp->A.max_u, s->wp->T.max_u, s->wp->A.max_rows, s->wp->T.max_rows,
                             s->wp->A.max_slices, s->wp->T.max_slices, s->wp->A.max_dict, s->wp->T.max_dict,
                             static_cast<unsigned long long>(s->wp->A.rec.bytes()),
                             static_cast<unsigned long long>(s->wp->T.rec.bytes()), s->win_smem_fista, s->win_smem_tau);
        }
    }
    if (!s->win)  // stream engine: Lanczos tau unless WBX_TAU=power (the window attempts may have reset it)
        s->tau_lanczos = sizeof(T) == 4 && !(std::getenv("WBX_TAU") && std::string(std::getenv("WBX_TAU")) == "power");
    // stencil engine for the FISTA iterations (fp32 single images; the operator carries its
    // generator groups): 2 then 1 CTA per SM
    const char* se = std::getenv("WBX_STENCIL");
    if (sizeof(T) == 4 && s->batch == 1 && s->op->has_gens && se && std::string(se) != "0" &&
        !(eng && std::string(eng) == "stream")) {
        for (int bps = 1; bps >= 1 && !s->stencil; --bps) {
            const uint32_t G = static_cast<uint32_t>(bps * s->ctx->num_sms);
            auto sp = stencil_plan_for(s->op, G, kStWarps, s->ctx->stream);
            std::string why;
            if (!stencil_plan_ok(*sp, &why)) {
                if (std::getenv("WBX_VERBOSE")) std::fprintf(stderr, "wbx stencil engine: G=%u: %s\n", G, why.c_str());
                continue;
            }
            const unsigned smem = st_smem_layout(view_of(*sp)).total;
            const unsigned limit = bps == 1 ? 220u * 1024u : (227u * 1024u) / bps - 2048u;
            if (std::getenv("WBX_VERBOSE"))
                std::fprintf(stderr, "wbx stencil engine: G=%u smem %u limit %u\n", G, smem, limit);
            if (smem > limit) continue;
            const void* k = reinterpret_cast<const void*>(fista_stencil_kernel);
            WBX_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            int occ = 0;
            WBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kStBlock, smem));
            if (occ < bps) continue;
            s->stencil = true;
            s->sp = sp;
            s->grid_st = static_cast<int>(G);
            s->st_smem = smem;
            s->yF.alloc(s->op->n);    // y (phase A source), natural layout
            s->resF.alloc(s->op->n);  // residual (phase T source)
        }
    }
}

}  // namespace

// The preconditioner / weight dependent state of a solver (its layouts, engines and buffers
// depend on the operator and the configuration only): used by setup and by a cached solver
// that is reused with new P, w (wbx_pgd)
void upload_pw(wbx_solver* s, const double* p, const double* w) {
    const wbx_op* op = s->op;
    const uint64_t n = op->n, nC = op->nC;
    cudaStream_t st = s->ctx->stream;
    for (uint64_t i = 0; i < n; ++i) {
        if (!(p[i] > 0.0)) fail(WBX_BAD_SPEC, "preconditioner entries must be strictly positive");
    }
    std::vector<double> hp(nC), hw(nC), hisp(nC);
    for (uint64_t c = 0; c < nC; ++c) {
        const uint32_t g = op->h_C_glob[c];
        hp[c] = p[g];
        hw[c] = w[g];
        hisp[c] = 1.0 / std::sqrt(p[g]);  // solver.cpp:72
    }
    s->pC.upload(hp, st);
    s->wC.upload(hw, st);
    s->ispC.upload(hisp, st);
    if (s->p_full.n != n) s->p_full.alloc(n);
    s->p_full.upload(p, n, st);
    if (s->w_full.n != n) s->w_full.alloc(n);
    s->w_full.upload(w, n, st);
}

// a cached solver (same operator and configuration) with a new P, w, lambda
void solver_update(wbx_solver* s, const double* p, const double* w, double lambda) {
    upload_pw(s, p, w);
    s->lambda = lambda;
    if (s->circ) {  // the block-Fourier estimate needs P constant on the column orbits
        std::string why;
        std::vector<double> isp;
        const bool was = s->tau_circ;
        s->tau_circ = circ_check_p(*s->circ, p, isp, &why);
        if (s->tau_circ) {
            s->circ_isp.upload(isp, s->ctx->stream);
            if (!s->circ_work.p) {
                s->circ_work.alloc(circ_work_doubles(*s->circ));
                WBX_CUDA(cudaMemsetAsync(s->circ_work.p, 0, s->circ_work.bytes(), s->ctx->stream));
            }
        }
        if (was != s->tau_circ && s->g_tau) {  // the step-estimate graph changes
            cudaGraphExecDestroy(s->g_tau);
            s->g_tau = nullptr;
        }
    }
    WBX_CUDA(cudaStreamSynchronize(s->ctx->stream));
}

void solver_setup(wbx_solver* s, const double* p, const double* w) {
    const wbx_op* op = s->op;
    const uint64_t nC = op->nC;
    cudaStream_t st = s->ctx->stream;
    upload_pw(s, p, w);
    const uint64_t K = s->cfg.max_iters;
    std::vector<double> b64(K > 0 ? K : 1, 0.0);
    std::vector<float> b32(K > 0 ? K : 1, 0.f);
    const bool momentum = s->accelerate && !s->cfg.zero_momentum;
    for (uint64_t k = 1; k <= K; ++k) {
        // solver.cpp:142-144
        const double beta =
            momentum ? (static_cast<double>(k) - 1.0) / (static_cast<double>(k) + 2.0) : 0.0;
        b64[k - 1] = beta;
        b32[k - 1] = static_cast<float>(beta);
    }
    s->beta64.upload(b64, st);
    s->beta32.upload(b32, st);
    if (s->cfg.precision == WBX_FP64)
        alloc_state<double>(s);
    else
        alloc_state<float>(s);
    s->dec_grid = 4 * s->ctx->num_sms;
    // step estimate: block-Fourier for translation-invariant operators on the fp32 hot path
    // (WBX_TAU=lanczos / power keep the full-operator estimates; the fp64 reference mode keeps
    // the literal power iteration, bitwise)
    const char* tau_env = std::getenv("WBX_TAU");
    if (s->cfg.precision == WBX_FP32 && (s->basis || op->has_layout) &&
        !(tau_env && (std::string(tau_env) == "lanczos" || std::string(tau_env) == "power"))) {
        auto plan = circ_plan_for(op, s->basis);
        std::string why, fwhy;
        std::vector<double> isp;
        const bool tau_on = !(tau_env && std::string(tau_env) == "spectral-off");
        const bool plan_ok = circ_plan_ok(*plan, &why, nullptr);
        if (plan_ok) {  // the G_f blocks serve both the estimate and the spectral engine
            circ_upload(*plan, st);
            s->circ = plan;
            s->circ_gram.alloc(circ_gram_doubles(*plan) / 2);
        }
        if (plan_ok && tau_on && circ_check_p(*plan, p, isp, &why)) {
            s->circ_isp.upload(isp, st);
            s->circ_work.alloc(circ_work_doubles(*plan));
            WBX_CUDA(cudaMemsetAsync(s->circ_work.p, 0, s->circ_work.bytes(), st));
            s->tau_circ = true;
        }
        // the spectral FISTA engine: single-image solves, with energy / support tracking too (solves
        // with the ref_energy stopping rule keep the window engine; WBX_ENGINE=window|stream and
        // WBX_STENCIL=1 select the others)
        const char* eng = std::getenv("WBX_ENGINE");
        const bool track_cfg = s->cfg.track_energy || s->cfg.track_support;
        if (!eng && !std::getenv("WBX_STENCIL") && !std::isfinite(s->cfg.ref_energy) &&
            !(track_cfg && s->cfg.max_iters == 0) &&  // (E(x0) alone: the window track kernel)
            circ_fista_ok(*plan, &fwhy) && static_cast<uint32_t>(s->ctx->num_sms) > circ_fista_blocks(*plan)) {
            // batches (C5, untracked): circ_slots images per launch, launches over the batch
            s->circ_slots = circ_fista_slots(*plan, s->ctx->num_sms, static_cast<uint32_t>(s->batch));
            s->circ_T.alloc(circ_exchange_doubles(*plan) / 2 * s->circ_slots);
            s->circ_counter.alloc(32 * s->circ_slots);
            if (track_cfg)
                s->circ_track.alloc(circ_track_doubles(*plan, static_cast<int>(s->cfg.max_iters), s->ctx->num_sms));
            s->fista_circ = true;
        }
        if (std::getenv("WBX_VERBOSE"))
            std::fprintf(stderr, "wbx: block-Fourier step estimate %s%s%s; spectral FISTA %s%s%s\n",
                         s->tau_circ ? "on" : "off", s->tau_circ ? "" : ": ", s->tau_circ ? "" : why.c_str(),
                         s->fista_circ ? "on" : "off", s->fista_circ ? "" : ": ", s->fista_circ ? "" : fwhy.c_str());
    }
    s->wv.alloc(nC ? nC : 1);
    s->uC.alloc(nC ? nC : 1);
    s->t64.alloc(op->nR ? op->nR : 1);
    s->out.alloc(OUT_COUNT);
    const uint64_t gmax = static_cast<uint64_t>(std::max({s->grid_fista, s->grid_tau, s->grid_tau_lz, s->grid_win, s->grid_st}));
    s->gen.alloc(kCounterWord + 32 * kMaxCounterGroups);
    s->arrive.alloc(gmax);
    s->part.alloc((2 * kRedSlots + 5) * gmax);  // barrier reductions + tracked window solve partials
    s->red.alloc(kRedSlots);
    WBX_CUDA(cudaMemsetAsync(s->gen.p, 0, s->gen.bytes(), st));
    WBX_CUDA(cudaMemsetAsync(s->arrive.p, 0, s->arrive.bytes(), st));
    const bool track = s->cfg.track_energy || s->cfg.track_support || std::isfinite(s->cfg.ref_energy);
    if (track && K > 0) {
        const uint64_t nwarps = static_cast<uint64_t>(s->dec_grid) * kBlock / 32;
        s->energies.alloc(K);
        s->supports.alloc(K);
        s->dec_reg.alloc(K);
        s->dec_supp.alloc(K);
        s->wreg.alloc(K * nwarps);
        s->wsup.alloc(K * nwarps);
    }
    if (std::getenv("WBX_TRACE_FILE")) {
        s->trace_cap = 1024;
        s->trace.alloc(s->trace_cap * gmax * 2);
        WBX_CUDA(cudaMemsetAsync(s->trace.p, 0, s->trace.bytes(), st));
    }
    WBX_CUDA(cudaEventCreate(&s->ev0));
    WBX_CUDA(cudaEventCreate(&s->ev1));
    WBX_CUDA(cudaEventCreate(&s->ev_mid));
    WBX_CUDA(cudaEventCreate(&s->ev_it0));
    WBX_CUDA(cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming));
    WBX_CUDA(cudaEventCreateWithFlags(&s->ev_an, cudaEventDisableTiming));
    WBX_CUDA(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
    WBX_CUDA(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    WBX_CUDA(cudaStreamCreateWithFlags(&s->aux_stream, cudaStreamNonBlocking));
    WBX_CUDA(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
    WBX_CUDA(cudaStreamSynchronize(st));
}

// Timing events: inside a captured graph they must be external event-record nodes (so the
// replay records them); outside a capture, plain records.
void record_event(cudaEvent_t ev, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    WBX_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive)
        WBX_CUDA(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal));
    else
        WBX_CUDA(cudaEventRecord(ev, st));
}

// Step estimate (independent of the image: it can run before the image is analysed, e.g.
// while the image is still being copied in) and the iterations, each bracketed by events.
void solver_tau(wbx_solver* s) {
    cudaStream_t st = s->ctx->stream;
    record_event(s->ev0, st);
    if (s->cfg.precision == WBX_FP64)
        run_tau<double>(s, s->x0full.p, s->xfull.p, st);
    else
        run_tau<float>(s, s->x0full.p, s->xfull.p, st);
    record_event(s->ev_mid, st);
}

void solver_iters(wbx_solver* s, const double* x0_full_dev, double* x_full_dev) {
    cudaStream_t st = s->ctx->stream;
    record_event(s->ev_it0, st);
    if (s->cfg.precision == WBX_FP64)
        run_iters<double>(s, x0_full_dev, x_full_dev, st);
    else
        run_iters<float>(s, x0_full_dev, x_full_dev, st);
    record_event(s->ev1, st);
}

void solver_run(wbx_solver* s, const double* x0_full_dev, double* x_full_dev) {
    solver_tau(s);
    solver_iters(s, x0_full_dev, x_full_dev);
}

float solve_ms_of(const wbx_solver* s) {  // tau + iterations (device events)
    float t = 0.f, i = 0.f;
    WBX_CUDA(cudaEventElapsedTime(&t, s->ev0, s->ev_mid));
    WBX_CUDA(cudaEventElapsedTime(&i, s->ev_it0, s->ev1));
    return t + i;
}

void solver_report(wbx_solver* s, wbx_report* rep) {
    cudaStream_t st = s->ctx->stream;
    double out[OUT_COUNT];
    WBX_CUDA(cudaMemcpyAsync(out, s->out.p, sizeof out, cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    ms = solve_ms_of(s);
    s->last_solve_ms = ms;
    if (s->trace.p) {
        if (FILE* f = std::fopen(std::getenv("WBX_TRACE_FILE"), "ab")) {
            std::vector<unsigned long long> h(s->trace.n);
            WBX_CUDA(cudaMemcpy(h.data(), s->trace.p, s->trace.bytes(), cudaMemcpyDeviceToHost));
            const unsigned long long hdr[2] = {static_cast<unsigned long long>(s->grid_fista), s->trace_cap};
            std::fwrite(hdr, sizeof hdr, 1, f);
            std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
            std::fclose(f);
        }
    }
    if (out[OUT_STATUS] == 8.0) fail(WBX_NONFINITE_ENERGY, "solver diverged (non-finite energy)");
    if (std::getenv("WBX_VERBOSE"))
        std::fprintf(stderr, "wbx tau: %.17g after %g reference iterations, %g operator product pairs (%s)\n",
                     out[OUT_TAU], out[OUT_TAU_ITERS], out[OUT_TAU_STEPS],
                     s->tau_circ ? "block-Fourier" : (s->tau_lanczos || s->tau_stream_lz) ? "lanczos" : "power");
    if (rep == nullptr) return;
    rep->iters_used = static_cast<uint64_t>(out[OUT_ITERS_USED]);
    rep->tau = out[OUT_TAU];
    rep->tau_iters = static_cast<uint32_t>(out[OUT_TAU_ITERS]);
    rep->initial_energy = out[OUT_INITIAL_ENERGY];
    rep->wall_time_s = ms * 1e-3;
    rep->ops_per_pixel_per_iter = 2.0 * static_cast<double>(s->op->nnz) / static_cast<double>(s->op->n);
    const uint64_t used = rep->iters_used;
    if (rep->energies && s->energies.p && used > 0)
        WBX_CUDA(cudaMemcpy(rep->energies, s->energies.p, used * sizeof(double), cudaMemcpyDeviceToHost));
    if (rep->support_sizes && s->supports.p && used > 0)
        WBX_CUDA(cudaMemcpy(rep->support_sizes, s->supports.p, used * sizeof(uint64_t), cudaMemcpyDeviceToHost));
}

void launch_clamp(wbx_ctx* ctx, double* u, uint64_t n, cudaStream_t st) {
    clamp_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(u, n);
    count_launch(ctx);
}

wbx_solver* solver_new(wbx_ctx* ctx, const wbx_op* op, wbx_basis* basis, double lambda,
                       const wbx_solver_cfg& cfg, int accelerate) {
    if (cfg.precision != WBX_FP32 && cfg.precision != WBX_FP64)
        fail(WBX_BAD_SPEC, "precision must be 32 or 64");
    if (cfg.max_iters > 0x7fffffffull) fail(WBX_TOO_LARGE, "max_iters too large");
    if (cfg.precision == WBX_FP32 && !(op->A.seg_ok && op->T.seg_ok))
        fail(WBX_TOO_LARGE, "operator rows longer than 496 nonzeros: fp32 layout unavailable, use precision 64");
    auto* s = new wbx_solver();
    s->ctx = ctx;
    s->op = op;
    s->basis = basis;
    s->n = op->n;
    s->lambda = lambda;
    s->cfg = cfg;
    s->accelerate = accelerate;
    return s;
}

void solver_free(wbx_solver* s) {
    if (!s) return;
    cudaStreamSynchronize(s->ctx->stream);
    if (s->ev0) cudaEventDestroy(s->ev0);
    if (s->ev1) cudaEventDestroy(s->ev1);
    if (s->ev_mid) cudaEventDestroy(s->ev_mid);
    if (s->ev_it0) cudaEventDestroy(s->ev_it0);
    if (s->ev_in) cudaEventDestroy(s->ev_in);
    if (s->ev_an) cudaEventDestroy(s->ev_an);
    if (s->ev_fork) cudaEventDestroy(s->ev_fork);
    if (s->ev_join) cudaEventDestroy(s->ev_join);
    if (s->aux_stream) cudaStreamDestroy(s->aux_stream);
    if (s->g_an) cudaGraphExecDestroy(s->g_an);
    if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
    if (s->g_tau) cudaGraphExecDestroy(s->g_tau);
    if (s->g_rest) cudaGraphExecDestroy(s->g_rest);
    delete s;
}

// wbx_pgd's solver cache: the reference calls fista() / ista() repeatedly on one operator; a
// solver's layouts, engines and device buffers depend on (context, operator, configuration,
// accelerate) only, so a repeated call re-uploads P, w and x0 instead of rebuilding it. A solver
// is taken out while in use; at most 4 are kept; entries of an operator are dropped when it is
// destroyed or its layout changes, entries of a context when it is destroyed.
namespace {
struct PgdEntry {
    wbx_ctx* ctx;
    const wbx_op* op;
    int accelerate;
    wbx_solver_cfg cfg;
    wbx_solver* s;
};
std::mutex g_pgd_mu;
std::list<PgdEntry> g_pgd;  // most recent first
constexpr size_t kPgdCache = 4;
}  // namespace

wbx_solver* pgd_acquire(wbx_ctx* ctx, const wbx_op* op, const wbx_solver_cfg& cfg, int accelerate, double lambda,
                        const double* p, const double* w) {
    wbx_solver* s = nullptr;
    {
        std::lock_guard<std::mutex> g(g_pgd_mu);
        for (auto it = g_pgd.begin(); it != g_pgd.end(); ++it)
            if (it->ctx == ctx && it->op == op && it->accelerate == accelerate &&
                std::memcmp(&it->cfg, &cfg, sizeof cfg) == 0) {
                s = it->s;
                g_pgd.erase(it);
                break;
            }
    }
    if (s) {
        try {
            solver_update(s, p, w, lambda);
        } catch (...) {
            solver_free(s);
            throw;
        }
        return s;
    }
    s = solver_new(ctx, op, nullptr, lambda, cfg, accelerate);
    try {
        solver_setup(s, p, w);
        s->x0full.alloc(op->n);
        s->xfull.alloc(op->n);
    } catch (...) {
        solver_free(s);
        throw;
    }
    return s;
}

void pgd_release(wbx_solver* s) {
    std::vector<wbx_solver*> evict;
    {
        std::lock_guard<std::mutex> g(g_pgd_mu);
        g_pgd.push_front(PgdEntry{s->ctx, s->op, s->accelerate, s->cfg, s});
        while (g_pgd.size() > kPgdCache) {
            evict.push_back(g_pgd.back().s);
            g_pgd.pop_back();
        }
    }
    for (wbx_solver* e : evict) solver_free(e);
}

void pgd_purge(const wbx_ctx* ctx, const wbx_op* op) {
    std::vector<wbx_solver*> evict;
    {
        std::lock_guard<std::mutex> g(g_pgd_mu);
        for (auto it = g_pgd.begin(); it != g_pgd.end();)
            if ((ctx && it->ctx == ctx) || (op && it->op == op)) {
                evict.push_back(it->s);
                it = g_pgd.erase(it);
            } else {
                ++it;
            }
    }
    for (wbx_solver* e : evict) solver_free(e);
}

double* solver_x0_buf(wbx_solver* s) { return s->x0full.p; }
double* solver_x_buf(wbx_solver* s) { return s->xfull.p; }

void solver_alloc_images(wbx_solver* s) {
    const uint64_t B = static_cast<uint64_t>(s->batch);
    s->u0.alloc(s->n * B);
    s->x0full.alloc(s->n * B);
    s->xfull.alloc(s->n * B);
    s->uout.alloc(s->n * B);
    if (B > 1) s->bwork.alloc(2 * s->n * B);  // the batched DWTs' work buffers
}

}  // namespace wbx

namespace {

// the analysis of the input (x0 = Psi^* u0): independent of the step estimate, so it runs on the
// side stream concurrently with it
void deblur_analyze(wbx_solver* s, const double* u0_dev, cudaStream_t side) {
    const uint64_t n = s->n, B = static_cast<uint64_t>(s->batch);
    if (B > 1)  // one launch per level pass for the whole batch
        wbx::analyze_dev_n(s->basis, u0_dev, s->x0full.p, static_cast<uint32_t>(B), s->bwork.p, s->bwork.p + B * n, side);
    else
        wbx::analyze_dev(s->basis, u0_dev, s->x0full.p, side);
}

// the rest of a deblur after the step estimate and the analysis: iterations -> synthesize (-> clamp)
void deblur_rest(wbx_solver* s, double* u_dev, int clamp, cudaStream_t st) {
    const uint64_t n = s->n, B = static_cast<uint64_t>(s->batch);
    wbx::solver_iters(s, s->x0full.p, s->xfull.p);
    if (B > 1)
        wbx::synthesize_dev_n(s->basis, s->xfull.p, u_dev, static_cast<uint32_t>(B), s->bwork.p, s->bwork.p + B * n, st,
                              clamp);
    else
        wbx::synthesize_dev(s->basis, s->xfull.p, u_dev, st, clamp);
}

// capture fn's enqueues on st into an executable graph; counts the kernels it enqueued
template <typename F>
cudaGraphExec_t capture_graph(wbx_solver* s, cudaStream_t st, uint64_t* launches, F fn) {
    const uint64_t before = s->ctx->launches;
    cudaGraph_t g = nullptr;
    WBX_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
        fn();
    } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    WBX_CUDA(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    WBX_CUDA(e);
    *launches = s->ctx->launches - before;
    s->ctx->launches = before;  // counted again at every replay
    return exec;
}

bool graphs_wanted(const wbx_solver* s) {
    static const bool off = std::getenv("WBX_GRAPH") && std::string(std::getenv("WBX_GRAPH")) == "0";
    return !off && !s->graphs_off && !s->trace.p;
}

}  // namespace

extern "C" {

int wbx_deblur_dev(wbx_solver* s, const double* u0_dev, double* u_dev, int clamp) {
    try {
        if (!s || !u0_dev || !u_dev) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_deblur_dev");
        cudaStream_t st = s->ctx->stream, side = s->copy_stream;
        const uint64_t before = s->ctx->launches;
        if (graphs_wanted(s)) {
            // three graphs: the image-independent step estimate on the main stream, concurrently
            // the analysis of the input on the side stream (after a pending host->device copy of
            // the image, queued there), then iterations + synthesis; ~25 launches -> 3
            try {
                if (!s->g_tau) s->g_tau = capture_graph(s, st, &s->g_tau_launches, [&] { wbx::solver_tau(s); });
                if (!s->g_an || s->g_an_u0 != u0_dev) {
                    if (s->g_an) cudaGraphExecDestroy(s->g_an);
                    s->g_an = nullptr;
                    s->g_an = capture_graph(s, side, &s->g_an_launches, [&] { deblur_analyze(s, u0_dev, side); });
                    s->g_an_u0 = u0_dev;
                }
                if (!s->g_rest || s->g_u != u_dev || s->g_clamp != clamp) {
                    if (s->g_rest) cudaGraphExecDestroy(s->g_rest);
                    s->g_rest = nullptr;
                    s->g_rest = capture_graph(s, st, &s->g_rest_launches, [&] { deblur_rest(s, u_dev, clamp, st); });
                    s->g_u = u_dev;
                    s->g_clamp = clamp;
                }
            } catch (const wbx::Error&) {  // capture not supported here: enqueue directly from now on
                cudaGetLastError();
                s->graphs_off = true;
            }
        }
        // the side stream starts after everything queued so far on the main stream (which may
        // still read x0full); a pending image copy is already queued on it
        if (!s->input_pending) {
            WBX_CUDA(cudaEventRecord(s->ev_in, st));
            WBX_CUDA(cudaStreamWaitEvent(side, s->ev_in, 0));
        }
        s->input_pending = false;
        if (graphs_wanted(s)) {
            WBX_CUDA(cudaGraphLaunch(s->g_an, side));
            WBX_CUDA(cudaEventRecord(s->ev_an, side));
            WBX_CUDA(cudaGraphLaunch(s->g_tau, st));
            WBX_CUDA(cudaStreamWaitEvent(st, s->ev_an, 0));
            WBX_CUDA(cudaGraphLaunch(s->g_rest, st));
            s->ctx->launches += s->g_tau_launches + s->g_an_launches + s->g_rest_launches;
        } else {
            deblur_analyze(s, u0_dev, side);
            WBX_CUDA(cudaEventRecord(s->ev_an, side));
            wbx::solver_tau(s);  // image-independent: concurrently with the copy and the analysis
            WBX_CUDA(cudaStreamWaitEvent(st, s->ev_an, 0));
            deblur_rest(s, u_dev, clamp, st);
        }
        WBX_CUDA(cudaGetLastError());
        s->last_launches = s->ctx->launches - before;
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_deblur(wbx_solver* s, const double* u0, double* u, int clamp, wbx_report* report) {
    try {
        if (!s || !u0 || !u) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_deblur");
        cudaStream_t st = s->ctx->stream;
        const uint64_t bytes = s->n * static_cast<uint64_t>(s->batch) * sizeof(double);
        // the image copy runs on a side stream (after everything queued so far, which may
        // still read s->u0) and overlaps the step estimate; the analysis waits for it
        WBX_CUDA(cudaEventRecord(s->ev_in, st));
        WBX_CUDA(cudaStreamWaitEvent(s->copy_stream, s->ev_in, 0));
        WBX_CUDA(cudaMemcpyAsync(s->u0.p, u0, bytes, cudaMemcpyHostToDevice, s->copy_stream));
        WBX_CUDA(cudaEventRecord(s->ev_in, s->copy_stream));
        s->input_pending = true;
        const int rc = wbx_deblur_dev(s, s->u0.p, s->uout.p, clamp);
        if (rc != WBX_OK) return rc;
        WBX_CUDA(cudaMemcpyAsync(u, s->uout.p, bytes, cudaMemcpyDeviceToHost, st));
        wbx::solver_report(s, report);  // synchronises
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_solver_last_stats(const wbx_solver* s, uint64_t* launches, float* solve_ms) {
    if (!s) return WBX_INVALID_ARGUMENT;
    if (launches) *launches = s->last_launches;
    if (solve_ms) {
        float ms = 0.f;
        float t = 0.f, i = 0.f;
        if (cudaEventElapsedTime(&t, s->ev0, s->ev_mid) != cudaSuccess ||
            cudaEventElapsedTime(&i, s->ev_it0, s->ev1) != cudaSuccess)
            return WBX_CUDA_ERROR;
        ms = t + i;
        *solve_ms = ms;
    }
    return WBX_OK;
}

int wbx_solver_phase_ms(const wbx_solver* s, float* tau_ms, float* iters_ms) {
    if (!s || !tau_ms || !iters_ms) return WBX_INVALID_ARGUMENT;
    if (cudaEventElapsedTime(tau_ms, s->ev0, s->ev_mid) != cudaSuccess) return WBX_CUDA_ERROR;
    if (cudaEventElapsedTime(iters_ms, s->ev_it0, s->ev1) != cudaSuccess) return WBX_CUDA_ERROR;
    return WBX_OK;
}

int wbx_solver_tau_stats(const wbx_solver* s, double* tau, uint32_t* ref_iters, uint32_t* product_pairs) {
    if (!s || !tau || !ref_iters || !product_pairs) return WBX_INVALID_ARGUMENT;
    double out[wbx::OUT_COUNT];
    // ordered after the solver kernels on the context's (non-blocking) stream
    if (cudaMemcpyAsync(out, s->out.p, sizeof out, cudaMemcpyDeviceToHost, s->ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(s->ctx->stream) != cudaSuccess)
        return WBX_CUDA_ERROR;
    *tau = out[wbx::OUT_TAU];
    *ref_iters = static_cast<uint32_t>(out[wbx::OUT_TAU_ITERS]);
    *product_pairs = static_cast<uint32_t>(out[wbx::OUT_TAU_STEPS]);
    return WBX_OK;
}

// Per-CTA features of the window layout of one side (0 = Theta rows, 1 = Theta^T rows), for
// fitting the balance cost model against traced phase times (tools/win_fit.py): out[G][6] =
// {rows, sum 1/m, sum nq/m, sum (q-1)/m, nonzeros, window entries}. Returns G in *G.
int wbx_diag_win_features(const wbx_solver* s, int side, double* out, int* G) {
    if (!s || !out || !G || !s->win || !s->wp) return WBX_INVALID_ARGUMENT;
    const wbx::WinSide& W = side ? s->wp->T : s->wp->A;
    const HostCompact& M = side ? s->op->hT : s->op->hA;
    std::vector<uint32_t> r_off(W.G + 1), u_off(W.G + 1);
    if (cudaMemcpy(r_off.data(), W.r_off.p, r_off.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(u_off.data(), W.u_off.p, u_off.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return WBX_CUDA_ERROR;
    for (uint32_t b = 0; b < W.G; ++b) {
        double f[6] = {0, 0, 0, 0, 0, static_cast<double>(u_off[b + 1] - u_off[b])};
        for (uint32_t r = r_off[b]; r < r_off[b + 1]; ++r) {
            const uint64_t len = M.ptr[r + 1] - M.ptr[r];
            const uint64_t q = std::max<uint64_t>(1, (len + wbx::kSegElems - 1) / wbx::kSegElems);
            const double m = static_cast<double>(32 / q), nq = static_cast<double>((len + q - 1) / q + 3) / 4.0;
            f[0] += 1.0;
            f[1] += 1.0 / m;
            f[2] += nq / m;
            f[3] += static_cast<double>(q - 1) / m;
            f[4] += static_cast<double>(len);
        }
        for (int k = 0; k < 6; ++k) out[b * 6 + k] = f[k];
    }
    *G = static_cast<int>(W.G);
    return WBX_OK;
}

int wbx_solver_kernels(const wbx_solver* s, char* buf, uint64_t len) {
    if (!s || !buf || len == 0) return WBX_INVALID_ARGUMENT;
    const bool fp64 = s->cfg.precision == WBX_FP64;
    const bool track = s->cfg.track_energy || s->cfg.track_support || std::isfinite(s->cfg.ref_energy);
    const char* tau = s->cfg.tau > 0.0 ? "set_tau_kernel"
                      : s->tau_circ ? "circ_lanczos_kernel"
                      : s->tau_stream_lz ? "tau_lanczos_kernel"
                      : s->win        ? (s->tau_lanczos ? "tau_lanczos_win_kernel" : "tau_win_kernel")
                      : (!fp64 && s->tau_lanczos) ? "tau_lanczos_kernel"
                                                   : (fp64 ? "tau_kernel<double>" : "tau_kernel<float>");
    const char* it = s->fista_circ                                  ? "circ_fista_kernel"
                     : (s->stencil && !track && s->batch == 1) ? "fista_stencil_kernel"
                     : (s->win && !track && s->batch == 1) ? "fista_win_kernel"
                     : (s->win_track && track && s->batch == 1) ? "fista_win_track_kernel"
                     : s->batch == 4                      ? "fista_batch_kernel<4>"
                     : s->batch == 8                      ? "fista_batch_kernel<8>"
                     : fp64                               ? "fista_kernel<double>"
                                                          : "fista_kernel<float>";
    std::snprintf(buf, len, "%s %s", tau, it);
    return WBX_OK;
}

}  // extern "C"

extern "C" int wbx_solver_create_batch(wbx_ctx* ctx, const wbx_op* op, const wbx_basis* basis, const double* p,
                                       const double* w, double lambda, const wbx_solver_cfg* cfg, int batch,
                                       wbx_solver** out) {
    wbx_solver* s = nullptr;
    try {
        if (!ctx || !op || !basis || !p || !w || !cfg || !out)
            wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_solver_create_batch");
        if (batch != 1 && batch != 4 && batch != 8) wbx::fail(WBX_BAD_SPEC, "batch must be 1, 4 or 8");
        if (basis->n != op->n) wbx::fail(WBX_SHAPE_MISMATCH, "operator and basis sizes differ");
        if (batch > 1 && (cfg->precision != WBX_FP32 || cfg->track_energy || cfg->track_support ||
                          std::isfinite(cfg->ref_energy)))
            wbx::fail(WBX_BAD_SPEC, "batched solves are fp32 with a fixed iteration count (no energy tracking)");
        s = wbx::solver_new(ctx, op, const_cast<wbx_basis*>(basis), lambda, *cfg, 1);
        s->batch = batch;
        wbx::solver_setup(s, p, w);
        wbx::solver_alloc_images(s);
        *out = s;
        return WBX_OK;
    } catch (const wbx::Error& e) {
        if (s) wbx::solver_free(s);
        wbx_set_last_error(e.what());
        return e.status;
    }
}

extern "C" int wbx_solver_batch(const wbx_solver* s) { return s ? s->batch : 0; }
