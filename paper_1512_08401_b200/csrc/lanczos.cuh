// Lanczos estimate of the reference's power-iteration step (solver.cpp:69-99): the power
// iteration on the Lanczos tridiagonal T_m and the convergence check shared by the
// persistent solver kernels (solver.cu) and the row-sharded path (shard.cu). See
// tau_lanczos_win_kernel in solver.cu for the derivation.
#pragma once

#include <cstdint>

namespace wbx {
namespace {

constexpr int kLzCap = 200;

// The power iteration on T_m from e1 (warp-wide; identical inputs in every CTA give
// identical results, so every CTA takes the same decision without communication).
// Element i lives in lane i & 31, register i >> 5. Returns lambda at the stopping
// iteration; *iters = the reference's iteration count; *zero = the zero-operator sentinel.
template <int K>  // K = ceil(m / 32) registers per lane
__device__ __forceinline__ double lz_power_on_T_k(const double* al, const double* be, int m, double r2, int* iters,
                                                  bool* zero) {
    // y = T^(2it) e1 / mu_2it: one pentadiagonal product by T^2 per iteration (one dependent
    // round of shuffles instead of two); mu_{2it+1}/mu_{2it} = (T y)_0 = alpha_0 + beta_1 y_1
    const int lane = threadIdx.x & 31;
    // T^2 coefficients are rebuilt from alpha / beta (shared memory) every iteration: the
    // check keeps only y and z in registers, so it does not crowd the phases' registers
    auto A = [&](int i) { return (i >= 0 && i < m) ? al[i] : 0.0; };
    auto B = [&](int i) { return (i > 0 && i < m) ? be[i] : 0.0; };  // T[i-1][i]
    double y[K];
#pragma unroll
    for (int k = 0; k < K; ++k) y[k] = lane + 32 * k == 0 ? 1.0 : 0.0;
    const double a0 = A(0), b1 = B(1);
    double lam_prev = 0.0;
    *zero = false;
    for (int it = 0; it < 200; ++it) {
        const double y1 = __shfl_sync(0xffffffffu, y[0], 1);
        const double lam = (it == 0 ? r2 : 1.0) * fma(b1, y1, a0);  // lambda_it (y_0 = 1)
        double z[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double u1 = __shfl_up_sync(0xffffffffu, y[k], 1), u2 = __shfl_up_sync(0xffffffffu, y[k], 2);
            double d1 = __shfl_down_sync(0xffffffffu, y[k], 1), d2 = __shfl_down_sync(0xffffffffu, y[k], 2);
            const double p31 = __shfl_sync(0xffffffffu, y[k > 0 ? k - 1 : 0], 31);
            const double p30 = __shfl_sync(0xffffffffu, y[k > 0 ? k - 1 : 0], 30);
            const double n0 = __shfl_sync(0xffffffffu, y[k + 1 < K ? k + 1 : k], 0);
            const double n1 = __shfl_sync(0xffffffffu, y[k + 1 < K ? k + 1 : k], 1);
            if (lane == 0) {
                u1 = k > 0 ? p31 : 0.0;
                u2 = k > 0 ? p30 : 0.0;
            }
            if (lane == 1) u2 = k > 0 ? p31 : 0.0;
            if (lane == 31) {
                d1 = k + 1 < K ? n0 : 0.0;
                d2 = k + 1 < K ? n1 : 0.0;
            }
            if (lane == 30) d2 = k + 1 < K ? n0 : 0.0;
            const int i = lane + 32 * k;
            const double am = A(i - 1), a_ = A(i), ap = A(i + 1);
            const double bm = B(i - 1), b_ = B(i), bp = B(i + 1), bpp = B(i + 2);
            const double d = fma(a_, a_, fma(b_, b_, bp * bp));  // (T^2)[i][i]
            const double e1 = bp * (a_ + ap);                     // (T^2)[i][i+1]
            const double e2 = bp * bpp;                           // (T^2)[i][i+2]
            const double l1 = b_ * (am + a_);                     // (T^2)[i][i-1]
            const double l2 = bm * b_;                            // (T^2)[i][i-2]
            z[k] = fma(l2, u2, fma(l1, u1, fma(d, y[k], fma(e1, d1, e2 * d2))));
        }
        const double even = __shfl_sync(0xffffffffu, z[0], 0);  // mu_{2it+2} / mu_{2it} = |M v_it|^2
        if (even == 0.0) {  // M v = 0: the reference's zero-operator sentinel (solver.cpp:89)
            *zero = true;
            *iters = it + 1;
            return lam;
        }
        if (it > 0 && fabs(lam - lam_prev) <= 1e-6 * fabs(lam)) {
            *iters = it + 1;
            return lam;
        }
        lam_prev = lam;
        const double inv = 1.0 / even;
#pragma unroll
        for (int k = 0; k < K; ++k) y[k] = z[k] * inv;
    }
    *iters = 200;
    return lam_prev;
}

__device__ double lz_power_on_T(const double* al, const double* be, int m, double r2, int* iters, bool* zero) {
    static_assert(kLzCap <= 7 * 32, "lz_power_on_T dispatch covers m <= 224");
    switch ((m + 31) / 32) {
        case 1: return lz_power_on_T_k<1>(al, be, m, r2, iters, zero);
        case 2: return lz_power_on_T_k<2>(al, be, m, r2, iters, zero);
        case 3: return lz_power_on_T_k<3>(al, be, m, r2, iters, zero);
        case 4: return lz_power_on_T_k<4>(al, be, m, r2, iters, zero);
        case 5: return lz_power_on_T_k<5>(al, be, m, r2, iters, zero);
        case 6: return lz_power_on_T_k<6>(al, be, m, r2, iters, zero);
        default: return lz_power_on_T_k<7>(al, be, m, r2, iters, zero);
    }
}

struct LzCtl {  // control state of tau_lanczos_win_kernel (shared memory, identical in every CTA)
    double alpha, beta, rb;  // alpha_j, beta_j, 1 / beta_j of the current step
    int breakdown;
    double r2, lambda, check_prev, tol;
    int stop_prev, iters, steps, zero, done, gap;
};

// Evaluate T_m (warp 0) and take the decision: `final` (the cap, a breakdown) or the
// zero-operator sentinel end the estimate; otherwise it ends when this check agrees with the
// previous one (same stopping index, lambda within ctl->tol). All threads of the CTA call it.
__device__ __noinline__ bool lz_check(const double* al, const double* be, int m, bool final, LzCtl* ctl) {
    // warp 0 evaluates T_m and warp 1 T_{m-gap} at the same time (the other warps idle): two
    // estimates per check, so the first check at which they agree ends the estimate
    __shared__ double lam1;
    __shared__ int its1;
    __syncthreads();  // alpha / beta of the last step are written
    const int w = threadIdx.x >> 5;
    const int m1 = m - ctl->gap;
    if (w == 1 && !final && m1 >= 1) {
        int its = 0;
        bool z = false;
        const double lam = lz_power_on_T(al, be, m1, ctl->r2, &its, &z);
        if ((threadIdx.x & 31) == 0) {
            lam1 = lam;
            its1 = z ? -1 : its;
        }
    }
    if (w == 0) {
        int its = 0;
        bool z = false;
        const double lam = lz_power_on_T(al, be, m, ctl->r2, &its, &z);
        if (threadIdx.x == 0) {
            ctl->lambda = lam;
            ctl->iters = its;
            ctl->zero = z;
            ctl->steps = m;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double lam = ctl->lambda;
        ctl->done = final || ctl->zero ||
                    (m1 >= 1 && its1 == ctl->iters && fabs(lam - lam1) <= ctl->tol * fabs(lam));
    }
    __syncthreads();
    return ctl->done != 0;
}

}  // namespace
}  // namespace wbx
