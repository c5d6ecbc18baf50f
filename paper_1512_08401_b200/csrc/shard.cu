// Row-sharded solve of ONE image across ranks (BASELINE config C4).
//
// The compacted coordinate sets of the single-GPU solver (R = nonempty rows of Theta,
// C = nonempty columns, both sorted by descending length exactly as op_build.cu) are cut
// into `world` contiguous ranges balanced by nonzeros. Rank p owns rows R_p of Theta and
// rows C_p of Theta^T (= columns C_p of Theta) and the coordinates C_p of x and y. Vectors
// that cross ranks live in PADDED global buffers (rank q's slice at q * max_range) so the
// exchange after each phase is one equal-size all-gather (NCCL over NVLink/NVSwitch, driven
// by the host; or nothing when the shards are emulated on one GPU and share the buffers):
//     phase A   res[R_p] = Theta[R_p, :] y - x0[R_p]         -> all-gather res
//     phase T   g = Theta^T[C_p, :] res; fused update on C_p  -> all-gather y
// No reductions cross ranks in FISTA, and every row is summed sequentially in element order by
// one lane of the row-per-lane layout wherever it lives, so a sharded solve is BITWISE the same
// for every world size (world 1 = this engine on one GPU; given tau). estimate_step needs two scalars per
// power iteration: each rank writes its block-ordered sums into its slot of a [world][2]
// buffer, the buffer is all-gathered, and every rank sums the slots in rank order on the
// device (deterministic for any world size) and updates the iteration state there. The host
// only enqueues: nothing in the power iteration synchronises with it.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>

#include "internal.hpp"
#include "lanczos.cuh"
#include "sell.cuh"

extern "C" void wbx_set_last_error(const char* msg);

struct wbx_shard {
    wbx_ctx* ctx = nullptr;
    uint32_t world = 1, rank = 0;
    uint64_t n = 0, nnz = 0, nR = 0, nC = 0;
    uint64_t rlo = 0, rhi = 0, clo = 0, chi = 0, maxR = 0, maxC = 0;
    wbx_sell A, T;                          // A: rows R_p (cols: padded C); T: rows C_p (cols: padded R)
    wbx::DevBuf<uint32_t> R_own, C_own;     // original indices of the owned rows / coordinates
    wbx::DevBuf<uint32_t> isC;              // global bitmask of nonempty columns (decoupled pass)
    // bound exchange buffers (device pointers owned by the caller)
    float* y_pad = nullptr;
    float* res_pad = nullptr;
    double* u_pad = nullptr;
    double* t_pad = nullptr;
    double* sums_pad = nullptr;  // [world][2] per-rank power-iteration sums (all-gathered)
    // owned state
    wbx::DevBuf<float> xp, x0R, tp, thr, beta;
    wbx::DevBuf<double> pC, wC, ispC, wv, p_full, w_full, part;
    wbx::DevBuf<double> pstate;  // power iteration: {nw_prev, lambda_prev, iterations, flag}
    wbx::DevBuf<double> qp, lz;  // Lanczos estimate: q_j-1 on C_p; alpha / beta / control (LzState)
    double lambda = 0.0, tau = 0.0;
    int max_iters = 0;
    uint64_t device_bytes = 0;
};

namespace wbx {
namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ bool bit_set(const uint32_t* m, uint64_t i) { return (m[i >> 5] >> (i & 31)) & 1u; }

__device__ __forceinline__ double rng_normal(uint64_t seed, uint64_t i) {
    auto at = [](uint64_t s, uint64_t k) {
        uint64_t z = s + 0x9e3779b97f4a7c15ull * (k + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    };
    auto u01 = [](uint64_t v) { return (static_cast<double>(v >> 11) + 0.5) * 0x1p-53; };
    const uint64_t m = i >> 1;
    const double u1 = u01(at(seed, 2 * m)), u2 = u01(at(seed, 2 * m + 1));
    const double r = sqrt(-2.0 * log(u1)), a = 2.0 * M_PI * u2;
    return (i & 1) ? r * sin(a) : r * cos(a);
}

struct ShardArgs {
    SellView A, T;
    uint32_t rank;
    uint64_t n, nR_own, nC_own, maxR, maxC;
    const uint32_t* R_own;
    const uint32_t* C_own;
    const uint32_t* isC;
    float* y_pad;
    float* res_pad;
    double* u_pad;
    double* t_pad;
    float* xp;
    float* x0R;
    float* tp;
    float* thr;
    const float* beta;
    const double* pC;
    const double* wC;
    const double* ispC;
    double* wv;
    const double* p_full;
    const double* w_full;
    double* part;
    double* sums_pad;
    double* pstate;
    double* qp;
    double* lz;
    uint32_t world;
    double lambda, tau;
};

ShardArgs args_of(wbx_shard* s) {
    ShardArgs a{};
    a.A = view_of(s->A);
    a.T = view_of(s->T);
    a.rank = s->rank;
    a.n = s->n;
    a.nR_own = s->rhi - s->rlo;
    a.nC_own = s->chi - s->clo;
    a.maxR = s->maxR;
    a.maxC = s->maxC;
    a.R_own = s->R_own.p;
    a.C_own = s->C_own.p;
    a.isC = s->isC.p;
    a.y_pad = s->y_pad;
    a.res_pad = s->res_pad;
    a.u_pad = s->u_pad;
    a.t_pad = s->t_pad;
    a.xp = s->xp.p;
    a.x0R = s->x0R.p;
    a.tp = s->tp.p;
    a.thr = s->thr.p;
    a.beta = s->beta.p;
    a.pC = s->pC.p;
    a.wC = s->wC.p;
    a.ispC = s->ispC.p;
    a.wv = s->wv.p;
    a.p_full = s->p_full.p;
    a.w_full = s->w_full.p;
    a.part = s->part.p;
    a.sums_pad = s->sums_pad;
    a.pstate = s->pstate.p;
    a.qp = s->qp.p;
    a.lz = s->lz.p;
    a.world = s->world;
    a.lambda = s->lambda;
    a.tau = s->tau;
    return a;
}

// One warp per slice of the row-per-lane fp32 layout (wbx_sell::rslice/rpk, op_build.cu), one
// lane per row, the row summed sequentially in element order (fma in ACC), grid-stride over the
// slices; whole warps in or out, no early return (block reductions follow). A row's sum does not
// depend on which rank or slice holds it, so every world size gives the same bits.
template <typename ACC, typename X, typename Epi>
__device__ __forceinline__ void slice_rows(const SellView& M, const X* __restrict__ x, Epi epi) {
    constexpr uint32_t H = 4;  // {val, col, val, col} pairs per step (16-B loads, 512 B per warp)
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < M.xslices; s += nw) {
        const uint2 meta = M.rslice[s];
        const uint32_t L = meta.y, np = L >> 1;
        const uint4* p = M.rpk + meta.x + lane;
        ACC acc = ACC(0);
        for (uint32_t h = 0; h < np; h += H) {
            uint4 e[H];
#pragma unroll
            for (uint32_t j = 0; j < H; ++j) e[j] = h + j < np ? __ldg(p + (h + j) * kWarp) : make_uint4(0, 0, 0, 0);
            X g[2 * H];
#pragma unroll
            for (uint32_t j = 0; j < H; ++j) {
                g[2 * j] = h + j < np ? x[e[j].y] : X(0);
                g[2 * j + 1] = h + j < np ? x[e[j].w] : X(0);
            }
#pragma unroll
            for (uint32_t j = 0; j < H; ++j) {
                if (h + j < np) {
                    acc = fma(static_cast<ACC>(__uint_as_float(e[j].x)), static_cast<ACC>(g[2 * j]), acc);
                    acc = fma(static_cast<ACC>(__uint_as_float(e[j].z)), static_cast<ACC>(g[2 * j + 1]), acc);
                }
            }
        }
        if (L & 1u) {
            const uint2 t = __ldg(reinterpret_cast<const uint2*>(M.rpk + meta.x + np * kWarp) + lane);
            acc = fma(static_cast<ACC>(__uint_as_float(t.x)), static_cast<ACC>(x[t.y]), acc);
        }
        const uint32_t r = s * kWarp + lane;
        if (r < M.rows) epi(r, acc);
    }
}

__global__ void init_kernel(ShardArgs a, const double* x0_full) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < a.nC_own) {
        const float v = static_cast<float>(x0_full[a.C_own[i]]);
        a.y_pad[a.rank * a.maxC + i] = v;
        a.xp[i] = v;
        a.tp[i] = static_cast<float>(a.tau / a.pC[i]);
        a.thr[i] = static_cast<float>(__ddiv_rn(__dmul_rn(__dmul_rn(a.tau, a.lambda), a.wC[i]), a.pC[i]));
    }
    if (i < a.nR_own) a.x0R[i] = static_cast<float>(x0_full[a.R_own[i]]);
}

__global__ void phase_a_kernel(ShardArgs a) {
    float* res = a.res_pad + a.rank * a.maxR;
    slice_rows<float, float>(a.A, a.y_pad, [&](uint32_t r, float acc) { res[r] = acc - a.x0R[r]; });
}

__global__ void phase_t_kernel(ShardArgs a, int k) {
    const float beta = a.beta[k - 1];
    float* y = a.y_pad + a.rank * a.maxC;
    slice_rows<float, float>(a.T, a.res_pad, [&](uint32_t c, float g) {
        const float z0 = fmaf(-a.tp[c], g, y[c]);
        const float t = fabsf(z0) - a.thr[c];
        const float xn = t > 0.f ? (z0 > 0.f ? t : -t) : 0.f;
        y[c] = fmaf(beta, xn - a.xp[c], xn);
        a.xp[c] = xn;
    });
}

// decoupled coordinates of this rank's slice of [0, n): prox + momentum in registers
__global__ void decoupled_kernel(ShardArgs a, uint64_t lo, uint64_t hi, int K, const double* x0_full,
                                 double* x_full) {
    const uint64_t i = lo + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= hi || bit_set(a.isC, i)) return;
    const double w = a.w_full[i];
    const float thr = static_cast<float>(__ddiv_rn(__dmul_rn(__dmul_rn(a.tau, a.lambda), w), a.p_full[i]));
    float x = static_cast<float>(x0_full[i]), xp = x, y = x;
    for (int k = 1; k <= K; ++k) {
        const float t = fabsf(y) - thr;
        const float xn = t > 0.f ? (y > 0.f ? t : -t) : 0.f;
        const bool fixed = xn == 0.f && xp == 0.f;
        y = fmaf(a.beta[k - 1], xn - xp, xn);
        xp = xn;
        x = xn;
        if (fixed) break;
    }
    x_full[i] = static_cast<double>(x);
}

__global__ void finalize_kernel(ShardArgs a, double* x_full) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < a.nC_own) x_full[a.C_own[i]] = static_cast<double>(a.xp[i]);
}

// ---- estimate_step pieces (fp64 vectors, fp32 operator values)
__global__ void power_init_kernel(ShardArgs a, uint64_t lo, uint64_t hi) {
    __shared__ double sm[kBlock / 32 + 1];
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nt = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    double s2 = 0.0;
    for (uint64_t i = lo + t; i < hi; i += nt) {
        const double v = rng_normal(0x5eedull, i);
        s2 += v * v;
    }
    for (uint64_t c = t; c < a.nC_own; c += nt) {
        const double v = rng_normal(0x5eedull, a.C_own[c]);
        a.wv[c] = v;
        a.u_pad[a.rank * a.maxC + c] = a.ispC[c] * v;
    }
    s2 = block_sum<kBlock>(s2, sm);
    if (threadIdx.x == 0) a.part[2 * blockIdx.x] = s2;
    if (threadIdx.x == 0) a.part[2 * blockIdx.x + 1] = 0.0;
}

// power-iteration state flags: 0 running, 1 converged, 2 zero operator, 3 iteration cap
__global__ void power_a_kernel(ShardArgs a) {
    if (a.pstate[3] != 0.0) return;  // stopped: the remaining enqueued iterations are no-ops
    const double inv = a.pstate[0];
    double* t = a.t_pad + a.rank * a.maxR;
    slice_rows<double, double>(a.A, a.u_pad, [&](uint32_t r, double acc) { t[r] = acc / inv; });
}

__global__ void power_t_kernel(ShardArgs a) {
    if (a.pstate[3] != 0.0) return;
    __shared__ double sm[kBlock / 32 + 1];
    const double inv = a.pstate[0];
    double pl = 0.0, pn = 0.0;
    double* u = a.u_pad + a.rank * a.maxC;
    slice_rows<double, double>(a.T, a.t_pad, [&](uint32_t c, double g) {
        const double w = g * a.ispC[c];
        const double v = a.wv[c] / inv;
        pl += v * w;
        pn += w * w;
        a.wv[c] = w;
        u[c] = a.ispC[c] * w;
    });
    pl = block_sum<kBlock>(pl, sm);
    pn = block_sum<kBlock>(pn, sm);
    if (threadIdx.x == 0) {
        a.part[2 * blockIdx.x] = pl;
        a.part[2 * blockIdx.x + 1] = pn;
    }
}

// this rank's sums: the block partials folded by one warp (lane-strided sums, then a fixed
// shuffle tree: deterministic) -> sums_pad[rank]
__device__ __forceinline__ void warp_rank_sums(const ShardArgs& a, unsigned blocks) {
    double s0 = 0.0, s1 = 0.0;
    for (unsigned i = threadIdx.x; i < blocks; i += 32) {
        s0 += a.part[2 * i];
        s1 += a.part[2 * i + 1];
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (threadIdx.x == 0) {
        a.sums_pad[2 * a.rank] = s0;
        a.sums_pad[2 * a.rank + 1] = s1;
    }
}

__global__ void rank_sums_kernel(ShardArgs a, unsigned blocks, int init) {
    if (!init && a.pstate[3] != 0.0) return;
    warp_rank_sums(a, blocks);
}

// stopping rule of estimate_step (solver.cpp:84-95) on the all-gathered sums, rank order
__global__ void power_update_kernel(ShardArgs a, int first) {
    if (threadIdx.x != 0) return;
    double* st = a.pstate;
    double s0 = 0.0, s1 = 0.0;
    for (uint32_t r = 0; r < a.world; ++r) {
        s0 += a.sums_pad[2 * r];
        s1 += a.sums_pad[2 * r + 1];
    }
    if (first) {
        st[0] = sqrt(s0);  // |v0|
        st[1] = 0.0;
        st[2] = 0.0;
        st[3] = 0.0;
        return;
    }
    if (st[3] != 0.0) return;
    const double lam = s0, nw = sqrt(s1);
    const double it = st[2] + 1.0;
    st[2] = it;
    if (nw == 0.0) {
        st[3] = 2.0;
        return;
    }
    if (it > 1.0 && fabs(lam - st[1]) <= 1e-6 * fabs(lam)) {
        st[1] = lam;
        st[3] = 1.0;
        return;
    }
    st[1] = lam;
    st[0] = nw;
    if (it >= 200.0) st[3] = 3.0;
}

unsigned blocks_for(uint64_t threads) { return static_cast<unsigned>(std::max<uint64_t>(1, (threads + kBlock - 1) / kBlock)); }

}  // namespace
// ---- estimate_step by Lanczos (solver.cu tau_lanczos_win_kernel; same steps, same checks)
// lz state: [0, kLzCap) alpha_j, [kLzCap, 2 kLzCap) beta_j, then the scalars below
enum : int { LZ_R2 = 2 * kLzCap, LZ_DONE, LZ_LAMBDA, LZ_ITERS, LZ_STEPS, LZ_ZERO, LZ_J, LZ_COUNT };

__global__ void lz_init_kernel(ShardArgs a, uint64_t lo, uint64_t hi) {
    __shared__ double sm[kBlock / 32 + 1];
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nt = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    double s2 = 0.0, sc = 0.0;
    for (uint64_t i = lo + t; i < hi; i += nt) {
        const double v = rng_normal(0x5eedull, i);
        s2 += v * v;
    }
    for (uint64_t c = t; c < a.nC_own; c += nt) {
        const double v = rng_normal(0x5eedull, a.C_own[c]);
        a.wv[c] = v;
        a.qp[c] = 0.0;
        a.y_pad[a.rank * a.maxC + c] = static_cast<float>(a.ispC[c] * v);
        sc += v * v;
    }
    s2 = block_sum<kBlock>(s2, sm);
    sc = block_sum<kBlock>(sc, sm);
    if (threadIdx.x == 0) {
        a.part[2 * blockIdx.x] = s2;
        a.part[2 * blockIdx.x + 1] = sc;
    }
}

// phase A_j: t' = Theta[R_p, :] P^-1/2 w_j, partial |t'|^2. The Lanczos vectors that cross
// ranks are fp32 (P^-1/2 w_j in y_pad, t' in res_pad: the FISTA buffers, idle during the
// estimate), as in the single-GPU fp32 estimators; w_j, q_j-1 and every sum stay fp64.
__global__ void lz_a_kernel(ShardArgs a) {
    if (a.lz[LZ_DONE] != 0.0) return;
    __shared__ double sm[kBlock / 32 + 1];
    float* t = a.res_pad + a.rank * a.maxR;
    double acc = 0.0;
    slice_rows<float, float>(a.A, a.y_pad, [&](uint32_t r, float v) {
        t[r] = v;
        acc += static_cast<double>(v) * static_cast<double>(v);
    });
    acc = block_sum<kBlock>(acc, sm);
    if (threadIdx.x == 0) {
        a.part[2 * blockIdx.x] = acc;
        a.part[2 * blockIdx.x + 1] = 0.0;
    }
}

// phase T_j: w_j+1 = M q_j - alpha_j q_j - beta_j q_j-1 on C_p, partial |w_j+1|^2
__global__ void lz_t_kernel(ShardArgs a) {
    if (a.lz[LZ_DONE] != 0.0) return;
    __shared__ double sm[kBlock / 32 + 1];
    const int j = static_cast<int>(a.lz[LZ_J]);
    const double alpha = a.lz[j], beta = a.lz[kLzCap + j], rb = 1.0 / beta;
    float* u = a.y_pad + a.rank * a.maxC;
    double acc = 0.0;
    slice_rows<float, float>(a.T, a.res_pad, [&](uint32_t c, float gf) {
        const double g = gf;
        const double z = a.ispC[c] * g * rb;  // (M q_j)_c
        const double q = a.wv[c] * rb;        // q_j
        const double wn = z - alpha * q - beta * a.qp[c];
        a.wv[c] = wn;
        a.qp[c] = q;
        u[c] = static_cast<float>(a.ispC[c] * wn);
        acc += wn * wn;
    });
    acc = block_sum<kBlock>(acc, sm);
    if (threadIdx.x == 0) {
        a.part[2 * blockIdx.x] = acc;
        a.part[2 * blockIdx.x + 1] = 0.0;
    }
}

__global__ void lz_rank_sums_kernel(ShardArgs a, unsigned blocks, int init) {
    if (!init && a.lz[LZ_DONE] != 0.0) return;
    warp_rank_sums(a, blocks);
}

// on the all-gathered sums (rank order, every rank alike): phase 0 starts the estimate,
// 1 takes alpha_j, 2 takes beta_j+1 and runs the scheduled check (two warps)
__global__ void lz_update_kernel(ShardArgs a, int phase, int first, int every, int gap, double tol) {
    __shared__ LzCtl ctl;
    __shared__ int check, final;
    double* lz = a.lz;
    if (threadIdx.x == 0) {
        check = final = 0;
        double s0 = 0.0, s1 = 0.0;
        for (uint32_t r = 0; r < a.world; ++r) {
            s0 += a.sums_pad[2 * r];
            s1 += a.sums_pad[2 * r + 1];
        }
        if (phase == 0) {
            lz[LZ_R2] = s1 / s0;
            lz[kLzCap] = sqrt(s1);
            lz[LZ_J] = 0.0;
            lz[LZ_LAMBDA] = lz[LZ_ITERS] = lz[LZ_STEPS] = 0.0;
            lz[LZ_ZERO] = lz[LZ_DONE] = !(sqrt(s1) > 0.0) ? 1.0 : 0.0;
        } else if (lz[LZ_DONE] == 0.0) {
            const int j = static_cast<int>(lz[LZ_J]);
            if (phase == 1) {
                const double beta = lz[kLzCap + j];
                lz[j] = s0 / (beta * beta);
            } else {
                const double bn = sqrt(s0);
                const int jn = j + 1;
                lz[LZ_J] = jn;
                if (jn < kLzCap) lz[kLzCap + jn] = bn;
                final = jn == kLzCap || !(bn > 1e-13 * (fabs(lz[j]) + lz[kLzCap + j]));  // cap / breakdown
                check = final || (jn >= first && (jn - first) % every == 0);
                ctl.r2 = lz[LZ_R2];
                ctl.gap = gap;
                ctl.tol = tol;
                ctl.done = 0;
            }
        }
    }
    __syncthreads();
    if (!check) return;
    const int m = static_cast<int>(lz[LZ_J]);
    if (lz_check(lz, lz + kLzCap, m, final != 0, &ctl) && threadIdx.x == 0) {
        lz[LZ_DONE] = 1.0;
        lz[LZ_LAMBDA] = ctl.lambda;
        lz[LZ_ITERS] = ctl.iters;
        lz[LZ_STEPS] = ctl.steps;
        lz[LZ_ZERO] = ctl.zero;
    }
}

}  // namespace wbx

using wbx::kBlock;

extern "C" {

int wbx_shard_create(wbx_ctx* ctx, uint64_t n, const uint64_t* rowptr, const uint32_t* col, const double* val,
                     uint32_t world, uint32_t rank, wbx_shard** out) {
    try {
        if (!ctx || !rowptr || !out) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_shard_create");
        if (world < 1 || rank >= world) wbx::fail(WBX_BAD_SPEC, "bad world / rank");
        if (rowptr[0] != 0) wbx::fail(WBX_SHAPE_MISMATCH, "inconsistent row offsets");
        const uint64_t nnz = rowptr[n];
        for (uint64_t r = 0; r < n; ++r) {
            if (rowptr[r] > rowptr[r + 1]) wbx::fail(WBX_SHAPE_MISMATCH, "row offsets not nondecreasing");
            for (uint64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
                if (col[k] >= n) wbx::fail(WBX_SHAPE_MISMATCH, "column index out of range");
                if (k > rowptr[r] && col[k] <= col[k - 1])
                    wbx::fail(WBX_SHAPE_MISMATCH, "columns not strictly increasing in a row");
            }
        }
        auto s = std::make_unique<wbx_shard>();
        s->ctx = ctx;
        s->world = world;
        s->rank = rank;
        s->n = n;
        s->nnz = nnz;
        // transpose (ascending original row within a column)
        std::vector<uint64_t> toff(n + 1, 0);
        for (uint64_t k = 0; k < nnz; ++k) ++toff[col[k] + 1];
        for (uint64_t i = 0; i < n; ++i) toff[i + 1] += toff[i];
        std::vector<uint32_t> trow(nnz);
        std::vector<double> tval(nnz);
        {
            std::vector<uint64_t> cur(toff.begin(), toff.end() - 1);
            for (uint64_t r = 0; r < n; ++r)
                for (uint64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
                    const uint64_t p = cur[col[k]]++;
                    trow[p] = static_cast<uint32_t>(r);
                    tval[p] = val[k];
                }
        }
        // global R, C in the single-GPU solver's order (op_build.cu)
        std::vector<uint32_t> R, C;
        for (uint64_t r = 0; r < n; ++r)
            if (rowptr[r + 1] > rowptr[r]) R.push_back(static_cast<uint32_t>(r));
        for (uint64_t c = 0; c < n; ++c)
            if (toff[c + 1] > toff[c]) C.push_back(static_cast<uint32_t>(c));
        std::stable_sort(R.begin(), R.end(), [&](uint32_t a, uint32_t b) {
            return rowptr[a + 1] - rowptr[a] > rowptr[b + 1] - rowptr[b];
        });
        std::stable_sort(C.begin(), C.end(),
                         [&](uint32_t a, uint32_t b) { return toff[a + 1] - toff[a] > toff[b + 1] - toff[b]; });
        s->nR = R.size();
        s->nC = C.size();
        // contiguous ranges balanced by nonzeros
        auto cut = [&](const std::vector<uint32_t>& ids, auto len) {
            std::vector<uint64_t> bounds(world + 1, ids.size());
            bounds[0] = 0;
            uint64_t total = 0;
            for (uint32_t id : ids) total += len(id);
            uint64_t acc = 0, q = 1;
            for (uint64_t i = 0; i < ids.size() && q < world; ++i) {
                acc += len(ids[i]);
                while (q < world && acc * world >= total * q) bounds[q++] = i + 1;
            }
            return bounds;
        };
        const auto rb = cut(R, [&](uint32_t r) { return rowptr[r + 1] - rowptr[r]; });
        const auto cb = cut(C, [&](uint32_t c) { return toff[c + 1] - toff[c]; });
        for (uint32_t q = 0; q < world; ++q) {
            s->maxR = std::max<uint64_t>(s->maxR, rb[q + 1] - rb[q]);
            s->maxC = std::max<uint64_t>(s->maxC, cb[q + 1] - cb[q]);
        }
        s->maxR = std::max<uint64_t>(s->maxR, 1);
        s->maxC = std::max<uint64_t>(s->maxC, 1);
        s->rlo = rb[rank];
        s->rhi = rb[rank + 1];
        s->clo = cb[rank];
        s->chi = cb[rank + 1];
        // padded global positions
        std::vector<uint32_t> rpad(n, 0xffffffffu), cpad(n, 0xffffffffu);
        for (uint32_t q = 0; q < world; ++q) {
            for (uint64_t i = rb[q]; i < rb[q + 1]; ++i) rpad[R[i]] = static_cast<uint32_t>(q * s->maxR + (i - rb[q]));
            for (uint64_t i = cb[q]; i < cb[q + 1]; ++i) cpad[C[i]] = static_cast<uint32_t>(q * s->maxC + (i - cb[q]));
        }
        if (static_cast<uint64_t>(world) * s->maxR > 0xffffffffull || static_cast<uint64_t>(world) * s->maxC > 0xffffffffull)
            wbx::fail(WBX_TOO_LARGE, "padded index space exceeds 32 bits");
        cudaStream_t st = ctx->stream;
        uint64_t bytes = 0;
        const uint64_t r0 = s->rlo, c0 = s->clo;
        wbx::build_sell(
            s->A, s->rhi - s->rlo, [&](uint64_t i) { return rowptr[R[r0 + i] + 1] - rowptr[R[r0 + i]]; },
            [&](uint64_t i, uint64_t j, uint32_t& c, double& v) {
                const uint64_t k = rowptr[R[r0 + i]] + j;
                c = cpad[col[k]];
                v = val[k];
            },
            st, bytes);
        wbx::build_sell(
            s->T, s->chi - s->clo, [&](uint64_t i) { return toff[C[c0 + i] + 1] - toff[C[c0 + i]]; },
            [&](uint64_t i, uint64_t j, uint32_t& c, double& v) {
                const uint64_t k = toff[C[c0 + i]] + j;
                c = rpad[trow[k]];
                v = tval[k];
            },
            st, bytes);
        std::vector<uint32_t> Rown(R.begin() + static_cast<long>(s->rlo), R.begin() + static_cast<long>(s->rhi));
        std::vector<uint32_t> Cown(C.begin() + static_cast<long>(s->clo), C.begin() + static_cast<long>(s->chi));
        if (Rown.empty()) Rown.push_back(0);
        if (Cown.empty()) Cown.push_back(0);
        s->R_own.upload(Rown, st);
        s->C_own.upload(Cown, st);
        std::vector<uint32_t> mask((n + 31) / 32, 0);
        for (uint32_t c : C) mask[c / 32] |= 1u << (c % 32);
        s->isC.upload(mask, st);
        WBX_CUDA(cudaStreamSynchronize(st));
        s->device_bytes = bytes;
        *out = s.release();
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

// Host-only: the partition wbx_shard_create uses (row/column range bounds per rank), for
// planning and for testing without a GPU. rbounds/cbounds: world + 1 entries each.
int wbx_shard_plan(uint64_t n, const uint64_t* rowptr, const uint32_t* col, uint32_t world, uint64_t* rbounds,
                   uint64_t* cbounds) {
    try {
        if (!rowptr || !rbounds || !cbounds || world < 1) wbx::fail(WBX_INVALID_ARGUMENT, "bad wbx_shard_plan args");
        const uint64_t nnz = rowptr[n];
        std::vector<uint64_t> clen(n, 0);
        for (uint64_t k = 0; k < nnz; ++k) {
            if (col[k] >= n) wbx::fail(WBX_SHAPE_MISMATCH, "column index out of range");
            ++clen[col[k]];
        }
        std::vector<uint32_t> R, C;
        for (uint64_t r = 0; r < n; ++r)
            if (rowptr[r + 1] > rowptr[r]) R.push_back(static_cast<uint32_t>(r));
        for (uint64_t c = 0; c < n; ++c)
            if (clen[c]) C.push_back(static_cast<uint32_t>(c));
        std::stable_sort(R.begin(), R.end(), [&](uint32_t a, uint32_t b) {
            return rowptr[a + 1] - rowptr[a] > rowptr[b + 1] - rowptr[b];
        });
        std::stable_sort(C.begin(), C.end(), [&](uint32_t a, uint32_t b) { return clen[a] > clen[b]; });
        auto cut = [&](const std::vector<uint32_t>& ids, auto len, uint64_t* bounds) {
            for (uint32_t q = 0; q <= world; ++q) bounds[q] = ids.size();
            bounds[0] = 0;
            uint64_t total = 0;
            for (uint32_t id : ids) total += len(id);
            uint64_t acc = 0, q = 1;
            for (uint64_t i = 0; i < ids.size() && q < world; ++i) {
                acc += len(ids[i]);
                while (q < world && acc * world >= total * q) bounds[q++] = i + 1;
            }
        };
        cut(R, [&](uint32_t r) { return rowptr[r + 1] - rowptr[r]; }, rbounds);
        cut(C, [&](uint32_t c) { return clen[c]; }, cbounds);
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_shard_destroy(wbx_shard* s) {
    if (s) {
        cudaStreamSynchronize(s->ctx->stream);
        delete s;
    }
    return WBX_OK;
}

int wbx_shard_get_info(const wbx_shard* s, uint64_t* info8) {
    if (!s || !info8) return WBX_INVALID_ARGUMENT;
    const uint64_t v[8] = {s->world, s->rank, s->rlo, s->rhi, s->clo, s->chi, s->maxR, s->maxC};
    std::copy(v, v + 8, info8);
    return WBX_OK;
}

int wbx_shard_bind(wbx_shard* s, float* y_pad, float* res_pad, double* u_pad, double* t_pad) {
    if (!s || !y_pad || !res_pad || !u_pad || !t_pad) return WBX_INVALID_ARGUMENT;
    s->y_pad = y_pad;
    s->res_pad = res_pad;
    s->u_pad = u_pad;
    s->t_pad = t_pad;
    return WBX_OK;
}

int wbx_shard_setup(wbx_shard* s, const double* p, const double* w, double lambda, int max_iters,
                    int accelerate) {
    try {
        if (!s || !p || !w) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_shard_setup");
        cudaStream_t st = s->ctx->stream;
        const uint64_t nC = std::max<uint64_t>(1, s->chi - s->clo);
        std::vector<uint32_t> Cown(nC);
        WBX_CUDA(cudaMemcpy(Cown.data(), s->C_own.p, nC * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        std::vector<double> hp(nC), hw(nC), hi(nC);
        for (uint64_t i = 0; i < nC; ++i) {
            hp[i] = p[Cown[i]];
            hw[i] = w[Cown[i]];
            if (!(hp[i] > 0.0)) wbx::fail(WBX_BAD_SPEC, "preconditioner entries must be strictly positive");
            hi[i] = 1.0 / std::sqrt(hp[i]);
        }
        s->pC.upload(hp, st);
        s->wC.upload(hw, st);
        s->ispC.upload(hi, st);
        s->p_full.alloc(s->n);
        s->p_full.upload(p, s->n, st);
        s->w_full.alloc(s->n);
        s->w_full.upload(w, s->n, st);
        std::vector<float> b(std::max(1, max_iters), 0.f);
        for (int k = 1; k <= max_iters; ++k)
            b[k - 1] = accelerate ? static_cast<float>((static_cast<double>(k) - 1.0) / (static_cast<double>(k) + 2.0)) : 0.f;
        s->beta.upload(b, st);
        s->xp.alloc(nC);
        s->tp.alloc(nC);
        s->thr.alloc(nC);
        s->wv.alloc(nC);
        s->x0R.alloc(std::max<uint64_t>(1, s->rhi - s->rlo));
        // per-block partials of the reductions: the phase kernels run one warp per slice (the
        // full grid of either side), init 2 CTAs per SM
        const uint64_t gmax = std::max<uint64_t>({wbx::blocks_for(uint64_t(s->A.xslices) * 32),
                                                  wbx::blocks_for(uint64_t(s->T.xslices) * 32),
                                                  2 * static_cast<uint64_t>(s->ctx->num_sms)});
        s->part.alloc(2 * gmax);
        s->lambda = lambda;
        s->max_iters = max_iters;
        WBX_CUDA(cudaStreamSynchronize(st));
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

// step 0: x0 -> owned state (needs tau), decoupled coordinates of this rank's index range
int wbx_shard_init(wbx_shard* s, double tau, const double* x0_full_dev, double* x_full_dev) {
    if (!s || !x0_full_dev || !x_full_dev || !s->y_pad) return WBX_INVALID_ARGUMENT;
    s->tau = tau;
    cudaStream_t st = s->ctx->stream;
    wbx::ShardArgs a = wbx::args_of(s);
    const uint64_t m = std::max(a.nC_own, a.nR_own);
    wbx::init_kernel<<<wbx::blocks_for(m), kBlock, 0, st>>>(a, x0_full_dev);
    const uint64_t lo = s->n * s->rank / s->world, hi = s->n * (s->rank + 1) / s->world;
    wbx::decoupled_kernel<<<wbx::blocks_for(hi - lo), kBlock, 0, st>>>(a, lo, hi, s->max_iters, x0_full_dev, x_full_dev);
    wbx::count_launch(s->ctx, 2);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

int wbx_shard_phase_a(wbx_shard* s) {
    if (!s) return WBX_INVALID_ARGUMENT;
    wbx::ShardArgs a = wbx::args_of(s);
    if (a.A.xslices) wbx::phase_a_kernel<<<wbx::blocks_for(uint64_t(a.A.xslices) * 32), kBlock, 0, s->ctx->stream>>>(a);
    wbx::count_launch(s->ctx);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

int wbx_shard_phase_t(wbx_shard* s, int k) {
    if (!s || k < 1 || k > s->max_iters) return WBX_INVALID_ARGUMENT;
    wbx::ShardArgs a = wbx::args_of(s);
    if (a.T.xslices) wbx::phase_t_kernel<<<wbx::blocks_for(uint64_t(a.T.xslices) * 32), kBlock, 0, s->ctx->stream>>>(a, k);
    wbx::count_launch(s->ctx);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

int wbx_shard_finalize(wbx_shard* s, double* x_full_dev) {
    if (!s || !x_full_dev) return WBX_INVALID_ARGUMENT;
    wbx::ShardArgs a = wbx::args_of(s);
    wbx::finalize_kernel<<<wbx::blocks_for(a.nC_own), kBlock, 0, s->ctx->stream>>>(a, x_full_dev);
    wbx::count_launch(s->ctx);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

// estimate_step, device-resident (see the header comment): begin -> [all-gather sums] ->
// update(first) -> repeat { step_a -> [all-gather t] -> step_t -> [all-gather sums] ->
// update -> [all-gather u] } -> result.
int wbx_shard_bind_power(wbx_shard* s, double* sums_pad) {
    if (!s || !sums_pad) return WBX_INVALID_ARGUMENT;
    s->sums_pad = sums_pad;
    if (!s->pstate.p) {
        try {
            s->pstate.alloc(4);
        } catch (const wbx::Error& e) {
            wbx_set_last_error(e.what());
            return e.status;
        }
    }
    return WBX_OK;
}

int wbx_shard_power_begin(wbx_shard* s) {
    if (!s || !s->u_pad || !s->sums_pad || !s->pstate.p) return WBX_INVALID_ARGUMENT;
    wbx::ShardArgs a = wbx::args_of(s);
    const unsigned blocks = 2 * static_cast<unsigned>(s->ctx->num_sms);
    if (2ull * blocks > s->part.n) return WBX_TOO_LARGE;
    const uint64_t lo = s->n * s->rank / s->world, hi = s->n * (s->rank + 1) / s->world;
    wbx::power_init_kernel<<<blocks, kBlock, 0, s->ctx->stream>>>(a, lo, hi);
    wbx::rank_sums_kernel<<<1, 32, 0, s->ctx->stream>>>(a, blocks, 1);
    wbx::count_launch(s->ctx, 2);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

int wbx_shard_power_update(wbx_shard* s, int first) {
    if (!s || !s->sums_pad || !s->pstate.p) return WBX_INVALID_ARGUMENT;
    wbx::power_update_kernel<<<1, 32, 0, s->ctx->stream>>>(wbx::args_of(s), first);
    wbx::count_launch(s->ctx);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

int wbx_shard_power_step_a(wbx_shard* s) {
    if (!s || !s->pstate.p) return WBX_INVALID_ARGUMENT;
    wbx::ShardArgs a = wbx::args_of(s);
    if (a.A.xslices) wbx::power_a_kernel<<<wbx::blocks_for(uint64_t(a.A.xslices) * 32), kBlock, 0, s->ctx->stream>>>(a);
    wbx::count_launch(s->ctx);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

int wbx_shard_power_step_t(wbx_shard* s) {
    if (!s || !s->sums_pad || !s->pstate.p) return WBX_INVALID_ARGUMENT;
    wbx::ShardArgs a = wbx::args_of(s);
    // a bounded grid (grid-stride over slices) keeps the partials few for the ordered sum
    const unsigned blocks = wbx::blocks_for(uint64_t(std::max<uint32_t>(a.T.xslices, 1)) * 32);
    if (2ull * blocks > s->part.n) return WBX_TOO_LARGE;
    if (a.T.xslices) {
        wbx::power_t_kernel<<<blocks, kBlock, 0, s->ctx->stream>>>(a);
    } else {
        cudaMemsetAsync(s->part.p, 0, 2 * blocks * sizeof(double), s->ctx->stream);
    }
    wbx::rank_sums_kernel<<<1, 32, 0, s->ctx->stream>>>(a, blocks, 0);
    wbx::count_launch(s->ctx, 2);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

int wbx_shard_power_result(wbx_shard* s, double step_safety, double* tau, uint32_t* iters) {
    if (!s || !tau || !iters || !s->pstate.p) return WBX_INVALID_ARGUMENT;
    double st[4];
    if (cudaMemcpyAsync(st, s->pstate.p, sizeof st, cudaMemcpyDeviceToHost, s->ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(s->ctx->stream) != cudaSuccess)
        return WBX_CUDA_ERROR;
    const bool zero = st[3] == 2.0;
    *iters = static_cast<uint32_t>(st[2]);
    *tau = (zero || st[1] <= 0.0) ? 1.0 : 1.0 / (st[1] * step_safety);  // solver.cpp:89,97
    return WBX_OK;
}


// estimate_step by Lanczos, device-resident like the power iteration above:
// lz_begin -> [all-gather sums] -> lz_update(0) -> repeat { lz_step_a -> [all-gather t, sums]
// -> lz_update(1) -> lz_step_t -> [all-gather sums, u] -> lz_update(2) } -> lz_result.
// lz_done (synchronising) lets the host stop enqueueing once the scheduled check agreed.
int wbx_shard_lz_begin(wbx_shard* s) {
    if (!s || !s->u_pad || !s->sums_pad) return WBX_INVALID_ARGUMENT;
    try {
        if (!s->lz.p) s->lz.alloc(wbx::LZ_COUNT);
        if (!s->qp.p) s->qp.alloc(std::max<uint64_t>(s->chi - s->clo, 1));
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
    wbx::ShardArgs a = wbx::args_of(s);
    const unsigned blocks = 2 * static_cast<unsigned>(s->ctx->num_sms);
    if (2ull * blocks > s->part.n) return WBX_TOO_LARGE;
    const uint64_t lo = s->n * s->rank / s->world, hi = s->n * (s->rank + 1) / s->world;
    cudaMemsetAsync(s->lz.p, 0, s->lz.bytes(), s->ctx->stream);
    wbx::lz_init_kernel<<<blocks, kBlock, 0, s->ctx->stream>>>(a, lo, hi);
    wbx::lz_rank_sums_kernel<<<1, 32, 0, s->ctx->stream>>>(a, blocks, 1);
    wbx::count_launch(s->ctx, 2);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

int wbx_shard_lz_update(wbx_shard* s, int phase, int first, int every, int gap) {
    if (!s || !s->sums_pad || !s->lz.p || phase < 0 || phase > 2 || first < 1 || every < 1 || gap < 1)
        return WBX_INVALID_ARGUMENT;
    // the single-GPU solver's agreement tolerance (WBX_LZ_TOL, solver.cu make_args)
    const double tol = std::getenv("WBX_LZ_TOL") ? std::atof(std::getenv("WBX_LZ_TOL")) : 1e-8;
    wbx::lz_update_kernel<<<1, 64, 0, s->ctx->stream>>>(wbx::args_of(s), phase, first, every, gap, tol);
    wbx::count_launch(s->ctx);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

static int lz_phase(wbx_shard* s, bool tside) {
    if (!s || !s->lz.p || !s->sums_pad) return WBX_INVALID_ARGUMENT;
    wbx::ShardArgs a = wbx::args_of(s);
    const wbx::SellView& M = tside ? a.T : a.A;
    const unsigned blocks = wbx::blocks_for(uint64_t(std::max<uint32_t>(M.xslices, 1)) * 32);
    if (2ull * blocks > s->part.n) return WBX_TOO_LARGE;
    if (M.xslices) {
        if (tside)
            wbx::lz_t_kernel<<<blocks, kBlock, 0, s->ctx->stream>>>(a);
        else
            wbx::lz_a_kernel<<<blocks, kBlock, 0, s->ctx->stream>>>(a);
    } else {
        cudaMemsetAsync(s->part.p, 0, 2 * blocks * sizeof(double), s->ctx->stream);
    }
    wbx::lz_rank_sums_kernel<<<1, 32, 0, s->ctx->stream>>>(a, blocks, 0);
    wbx::count_launch(s->ctx, 2);
    return cudaGetLastError() == cudaSuccess ? WBX_OK : WBX_CUDA_ERROR;
}

int wbx_shard_lz_step_a(wbx_shard* s) { return lz_phase(s, false); }
int wbx_shard_lz_step_t(wbx_shard* s) { return lz_phase(s, true); }

int wbx_shard_lz_done(wbx_shard* s, int* done) {
    if (!s || !done || !s->lz.p) return WBX_INVALID_ARGUMENT;
    double d = 0.0;
    if (cudaMemcpyAsync(&d, s->lz.p + wbx::LZ_DONE, sizeof d, cudaMemcpyDeviceToHost, s->ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(s->ctx->stream) != cudaSuccess)
        return WBX_CUDA_ERROR;
    *done = d != 0.0;
    return WBX_OK;
}

int wbx_shard_lz_result(wbx_shard* s, double step_safety, double* tau, uint32_t* iters, uint32_t* steps) {
    if (!s || !tau || !iters || !steps || !s->lz.p) return WBX_INVALID_ARGUMENT;
    double st[wbx::LZ_COUNT];
    if (cudaMemcpyAsync(st, s->lz.p, sizeof st, cudaMemcpyDeviceToHost, s->ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(s->ctx->stream) != cudaSuccess)
        return WBX_CUDA_ERROR;
    if (st[wbx::LZ_DONE] == 0.0) {
        wbx_set_last_error("wbx_shard_lz_result: the estimate has not finished");
        return WBX_BAD_SPEC;
    }
    const double lam = st[wbx::LZ_LAMBDA];
    *iters = static_cast<uint32_t>(st[wbx::LZ_ITERS]);
    *steps = static_cast<uint32_t>(st[wbx::LZ_STEPS]);
    *tau = (st[wbx::LZ_ZERO] != 0.0 || lam <= 0.0) ? 1.0 : 1.0 / (lam * step_safety);  // solver.cpp:89,97
    return WBX_OK;
}

}  // extern "C"

// ====================================================================================== //
// The whole row-sharded deblur behind the C ABI (wbx_sharded_*): the host loop, the exchange
// (NCCL over NVLink, opened at run time, or nothing when every shard lives in this process),
// and a CUDA graph of the 100 FISTA iterations (phase kernels + all-gathers), so a solve is one
// host call after the first. estimate_step runs as graphs of kLzChunk Lanczos steps; the host
// reads the device's done flag once per chunk from the first scheduled check on.
#include <dlfcn.h>

#include "nccl.h"

namespace wbx {
namespace {

struct NcclApi {  // the NCCL entry points used here, resolved at run time (no link dependency)
    void* lib = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        // the NCCL already in the process (e.g. torch's) first, else the system's
        a.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!a.lib) a.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!a.lib) a.lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!a.lib) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.lib, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.lib, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.lib, "ncclCommDestroy"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.lib, "ncclAllGather"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(a.lib, "ncclAllReduce"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.lib, "ncclGetErrorString"));
        return a;
    }();
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.all_reduce || !api.comm_destroy)
        fail(WBX_CUDA_ERROR, "NCCL (libnccl.so.2) is not available");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(WBX_CUDA_ERROR, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

constexpr int kLzChunk = 4;  // Lanczos steps per captured graph (= the check period)

}  // namespace
}  // namespace wbx

struct wbx_comm {
    wbx_ctx* ctx = nullptr;
    uint32_t world = 1, rank = 0;
    ncclComm_t comm = nullptr;
};

struct wbx_sharded {
    wbx_ctx* ctx = nullptr;
    wbx_basis* basis = nullptr;
    wbx_comm* comm = nullptr;  // NULL: every shard in this process (emulation / one GPU)
    uint32_t world = 1;
    std::vector<wbx_shard*> shards;
    uint64_t n = 0, maxR = 0, maxC = 0;
    wbx::DevBuf<float> y, res;
    wbx::DevBuf<double> u, t, sums, x0, x;
    wbx_solver_cfg cfg{};
    int lz_first = 48, lz_every = 4, lz_gap = 4;
    bool power = false;
    cudaGraphExec_t fista_exec = nullptr, lz_exec = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    double tau = 0.0;
    uint32_t tau_iters = 0, tau_steps = 0;
    uint64_t last_launches = 0;
    ~wbx_sharded() {
        if (fista_exec) cudaGraphExecDestroy(fista_exec);
        if (lz_exec) cudaGraphExecDestroy(lz_exec);
        for (wbx_shard* s : shards) delete s;
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (ev2) cudaEventDestroy(ev2);
    }
};

namespace wbx {
namespace {

// In-place all-gather of the equal per-rank slices of a padded buffer (count elements each).
template <typename T>
void gather(wbx_sharded* S, T* buf, uint64_t count) {
    if (!S->comm || S->world == 1) return;  // shards in this process share the buffers
    const ncclDataType_t dt = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
    nccl_check(nccl().all_gather(buf + S->comm->rank * count, buf, count, dt, S->comm->comm, S->ctx->stream),
               "ncclAllGather");
}

void each(wbx_sharded* S, int (*fn)(wbx_shard*)) {
    for (wbx_shard* s : S->shards) {
        const int st = fn(s);
        if (st != WBX_OK) fail(st, std::string("shard step failed: ") + wbx_last_error());
    }
}

// FISTA iterations (phase A, all-gather res, phase T(k), all-gather y), k = 1..iters
void enqueue_fista(wbx_sharded* S) {
    for (int k = 1; k <= static_cast<int>(S->cfg.max_iters); ++k) {
        each(S, wbx_shard_phase_a);
        gather(S, S->res.p, S->maxR);
        for (wbx_shard* s : S->shards)
            if (wbx_shard_phase_t(s, k) != WBX_OK) fail(WBX_CUDA_ERROR, "phase T failed");
        gather(S, S->y.p, S->maxC);
    }
}

// kLzChunk Lanczos steps (no-ops on the device once the estimate is done)
void enqueue_lz_chunk(wbx_sharded* S) {
    auto update = [&](int phase) {
        for (wbx_shard* s : S->shards)
            if (wbx_shard_lz_update(s, phase, S->lz_first, S->lz_every, S->lz_gap) != WBX_OK)
                fail(WBX_CUDA_ERROR, "lz_update failed");
    };
    for (int j = 0; j < kLzChunk; ++j) {  // t' in res, P^-1/2 w in y (fp32)
        each(S, wbx_shard_lz_step_a);
        gather(S, S->res.p, S->maxR);
        gather(S, S->sums.p, 2);
        update(1);
        each(S, wbx_shard_lz_step_t);
        gather(S, S->sums.p, 2);
        gather(S, S->y.p, S->maxC);
        update(2);
    }
}

// capture fn's enqueues on the context stream into an executable graph (once)
template <typename F>
cudaGraphExec_t capture(wbx_sharded* S, F fn) {
    cudaStream_t st = S->ctx->stream;
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
    return exec;
}

bool graphs_enabled() {
    const char* e = std::getenv("WBX_SHARD_GRAPH");
    return !(e && std::string(e) == "0");
}

double estimate(wbx_sharded* S, double step_safety, uint32_t* iters, uint32_t* steps) {
    cudaStream_t st = S->ctx->stream;
    if (S->power) {  // the literal power iteration (WBX_TAU=power): fixed 200-step schedule
        each(S, wbx_shard_power_begin);
        gather(S, S->sums.p, 2);
        for (wbx_shard* s : S->shards) wbx_shard_power_update(s, 1);
        gather(S, S->u.p, S->maxC);
        for (int it = 0; it < 200; ++it) {
            each(S, wbx_shard_power_step_a);
            gather(S, S->t.p, S->maxR);
            each(S, wbx_shard_power_step_t);
            gather(S, S->sums.p, 2);
            for (wbx_shard* s : S->shards) wbx_shard_power_update(s, 0);
            gather(S, S->u.p, S->maxC);
        }
        double tau = 0.0;
        if (wbx_shard_power_result(S->shards[0], step_safety, &tau, iters) != WBX_OK)
            fail(WBX_CUDA_ERROR, "power result failed");
        *steps = *iters;
        return tau;
    }
    each(S, wbx_shard_lz_begin);
    gather(S, S->sums.p, 2);
    for (wbx_shard* s : S->shards) wbx_shard_lz_update(s, 0, S->lz_first, S->lz_every, S->lz_gap);
    gather(S, S->y.p, S->maxC);
    const bool graphs = graphs_enabled();
    if (graphs && !S->lz_exec) S->lz_exec = capture(S, [&] { enqueue_lz_chunk(S); });
    for (int j = 0; j < kLzCap; j += kLzChunk) {
        if (graphs) {
            WBX_CUDA(cudaGraphLaunch(S->lz_exec, st));
            count_launch(S->ctx, static_cast<uint64_t>(kLzChunk) * 6 * S->shards.size());
        } else {
            enqueue_lz_chunk(S);
        }
        const int done_j = j + kLzChunk;
        if (done_j >= S->lz_first || done_j >= kLzCap) {  // a check ran in this chunk (or the cap)
            int done = 0;
            if (wbx_shard_lz_done(S->shards[0], &done) != WBX_OK) fail(WBX_CUDA_ERROR, "lz_done failed");
            if (done) break;
        }
    }
    double tau = 0.0;
    if (wbx_shard_lz_result(S->shards[0], step_safety, &tau, iters, steps) != WBX_OK)
        fail(WBX_CUDA_ERROR, std::string("Lanczos result: ") + wbx_last_error());
    return tau;
}

__global__ void clamp01_kernel(double* u, uint64_t n) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) u[i] = fmin(fmax(u[i], 0.0), 1.0);  // std::clamp(v, 0, 1), waveblur.cpp:297
}

}  // namespace
}  // namespace wbx

extern "C" {

int wbx_comm_get_unique_id(uint8_t* id128) {
    try {
        if (!id128) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_comm_get_unique_id");
        ncclUniqueId id;
        wbx::nccl_check(wbx::nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(id128, id.internal, NCCL_UNIQUE_ID_BYTES);
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_comm_create(wbx_ctx* ctx, uint32_t world, uint32_t rank, const uint8_t* id128, wbx_comm** out) {
    try {
        if (!ctx || !id128 || !out) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_comm_create");
        if (world < 1 || rank >= world) wbx::fail(WBX_BAD_SPEC, "bad world / rank");
        auto c = std::make_unique<wbx_comm>();
        c->ctx = ctx;
        c->world = world;
        c->rank = rank;
        ncclUniqueId id;
        std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
        WBX_CUDA(cudaSetDevice(ctx->device));
        wbx::nccl_check(wbx::nccl().comm_init_rank(&c->comm, static_cast<int>(world), id, static_cast<int>(rank)),
                        "ncclCommInitRank");
        *out = c.release();
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_comm_destroy(wbx_comm* c) {
    if (!c) return WBX_OK;
    if (c->comm) wbx::nccl().comm_destroy(c->comm);
    delete c;
    return WBX_OK;
}

int wbx_sharded_create(wbx_ctx* ctx, uint64_t n, const uint64_t* rowptr, const uint32_t* col, const double* val,
                       wbx_basis* basis, const double* p, const double* w, double lambda, const wbx_solver_cfg* cfg,
                       uint32_t world, const uint32_t* ranks, uint32_t nranks, wbx_comm* comm, wbx_sharded** out) {
    try {
        if (!ctx || !rowptr || !basis || !p || !w || !cfg || !ranks || !out)
            wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_sharded_create");
        if (basis->n != n) wbx::fail(WBX_SHAPE_MISMATCH, "operator and basis sizes differ");
        if (cfg->precision != WBX_FP32 || cfg->track_energy || cfg->track_support || std::isfinite(cfg->ref_energy))
            wbx::fail(WBX_BAD_SPEC, "sharded solves are fp32 with a fixed iteration count (no energy tracking)");
        if (comm) {
            if (nranks != 1 || comm->world != world || ranks[0] != comm->rank)
                wbx::fail(WBX_BAD_SPEC, "a communicator run holds exactly its own rank");
        } else if (nranks != world) {
            wbx::fail(WBX_BAD_SPEC, "without a communicator every rank must live in this process");
        }
        auto S = std::make_unique<wbx_sharded>();
        S->ctx = ctx;
        S->basis = basis;
        S->comm = comm;
        S->world = world;
        S->n = n;
        S->cfg = *cfg;
        auto env = [](const char* k, int d) {
            const char* e = std::getenv(k);
            return e ? std::max(1, std::min(wbx::kLzCap, std::atoi(e))) : d;
        };
        S->lz_first = env("WBX_LZ_FIRST", 48);
        S->lz_every = wbx::kLzChunk;
        S->lz_gap = env("WBX_LZ_GAP", 4);
        S->power = std::getenv("WBX_TAU") && std::string(std::getenv("WBX_TAU")) == "power";
        for (uint32_t i = 0; i < nranks; ++i) {
            wbx_shard* sh = nullptr;
            const int st = wbx_shard_create(ctx, n, rowptr, col, val, world, ranks[i], &sh);
            if (st != WBX_OK) wbx::fail(st, wbx_last_error());
            S->shards.push_back(sh);
        }
        S->maxR = S->shards[0]->maxR;
        S->maxC = S->shards[0]->maxC;
        S->y.alloc(world * S->maxC);
        S->res.alloc(world * S->maxR);
        S->u.alloc(world * S->maxC);
        S->t.alloc(world * S->maxR);
        S->sums.alloc(2 * world);
        S->x0.alloc(n);
        S->x.alloc(n);
        cudaStream_t st = ctx->stream;
        WBX_CUDA(cudaMemsetAsync(S->y.p, 0, S->y.bytes(), st));
        WBX_CUDA(cudaMemsetAsync(S->res.p, 0, S->res.bytes(), st));
        WBX_CUDA(cudaMemsetAsync(S->u.p, 0, S->u.bytes(), st));
        WBX_CUDA(cudaMemsetAsync(S->t.p, 0, S->t.bytes(), st));
        for (wbx_shard* sh : S->shards) {
            wbx_shard_bind(sh, S->y.p, S->res.p, S->u.p, S->t.p);
            const int r = wbx_shard_setup(sh, p, w, lambda, static_cast<int>(cfg->max_iters), 1);
            if (r != WBX_OK) wbx::fail(r, wbx_last_error());
            wbx_shard_bind_power(sh, S->sums.p);
        }
        WBX_CUDA(cudaEventCreate(&S->ev0));
        WBX_CUDA(cudaEventCreate(&S->ev1));
        WBX_CUDA(cudaEventCreate(&S->ev2));
        WBX_CUDA(cudaStreamSynchronize(st));
        *out = S.release();
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_sharded_destroy(wbx_sharded* s) {
    if (s) {
        cudaStreamSynchronize(s->ctx->stream);
        delete s;
    }
    return WBX_OK;
}

int wbx_sharded_estimate_step(wbx_sharded* s, double step_safety, double* tau, uint32_t* iters, uint32_t* steps) {
    try {
        if (!s || !tau || !iters || !steps) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_sharded_estimate_step");
        *tau = wbx::estimate(s, step_safety, iters, steps);
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_sharded_deblur_dev(wbx_sharded* s, const double* u0_dev, double* u_dev, int clamp) {
    try {
        if (!s || !u0_dev || !u_dev) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_sharded_deblur_dev");
        cudaStream_t st = s->ctx->stream;
        const uint64_t before = s->ctx->launches;
        WBX_CUDA(cudaEventRecord(s->ev0, st));
        // every rank analyses the whole observation (x0 = Psi^* u0; bitwise the reference's)
        wbx::analyze_dev(s->basis, u0_dev, s->x0.p, st);
        double tau = s->cfg.tau;
        if (!(tau > 0.0)) tau = wbx::estimate(s, s->cfg.step_safety, &s->tau_iters, &s->tau_steps);
        s->tau = tau;
        WBX_CUDA(cudaEventRecord(s->ev1, st));
        WBX_CUDA(cudaMemsetAsync(s->x.p, 0, s->n * sizeof(double), st));
        for (wbx_shard* sh : s->shards)
            if (wbx_shard_init(sh, tau, s->x0.p, s->x.p) != WBX_OK) wbx::fail(WBX_CUDA_ERROR, "shard init failed");
        wbx::gather(s, s->y.p, s->maxC);
        if (wbx::graphs_enabled()) {
            if (!s->fista_exec) s->fista_exec = wbx::capture(s, [&] { wbx::enqueue_fista(s); });
            WBX_CUDA(cudaGraphLaunch(s->fista_exec, st));
            wbx::count_launch(s->ctx, 2 * s->cfg.max_iters * s->shards.size());
        } else {
            wbx::enqueue_fista(s);
        }
        for (wbx_shard* sh : s->shards)
            if (wbx_shard_finalize(sh, s->x.p) != WBX_OK) wbx::fail(WBX_CUDA_ERROR, "shard finalize failed");
        if (s->comm && s->world > 1)  // disjoint pieces (every other entry 0.0): the sum is exact
            wbx::nccl_check(wbx::nccl().all_reduce(s->x.p, s->x.p, s->n, ncclFloat64, ncclSum, s->comm->comm, st),
                            "ncclAllReduce");
        wbx::synthesize_dev(s->basis, s->x.p, u_dev, st);
        if (clamp) {
            wbx::clamp01_kernel<<<static_cast<unsigned>((s->n + 255) / 256), 256, 0, st>>>(u_dev, s->n);
            wbx::count_launch(s->ctx);
        }
        WBX_CUDA(cudaEventRecord(s->ev2, st));
        WBX_CUDA(cudaGetLastError());
        s->last_launches = s->ctx->launches - before;
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_sharded_stats(const wbx_sharded* s, double* tau, uint32_t* tau_iters, uint32_t* tau_steps, float* tau_ms,
                      float* iters_ms, uint64_t* launches) {
    if (!s) return WBX_INVALID_ARGUMENT;
    if (tau) *tau = s->tau;
    if (tau_iters) *tau_iters = s->tau_iters;
    if (tau_steps) *tau_steps = s->tau_steps;
    if (launches) *launches = s->last_launches;
    if (tau_ms && cudaEventElapsedTime(tau_ms, s->ev0, s->ev1) != cudaSuccess) return WBX_CUDA_ERROR;
    if (iters_ms && cudaEventElapsedTime(iters_ms, s->ev1, s->ev2) != cudaSuccess) return WBX_CUDA_ERROR;
    return WBX_OK;
}

}  // extern "C"
