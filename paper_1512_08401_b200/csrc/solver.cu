// Preconditioned FISTA / ISTA on the device: ONE persistent cooperative kernel per solve.
//
// Replaces run_pgd (`proj/src/solver.cpp:103-157`), estimate_step (:69-99) and
// prox_weighted_l1_P (:57-67). Per iteration the reference does 3 CSR SpMVs and ~6
// serial O(n) passes with fresh allocations; here one iteration is two grid-wide
// phases of one resident kernel:
//   phase A (rows R of Theta):      res[r] = (Theta y)[r] - x0[r]
//   ---- grid barrier ----
//   phase T (rows C of Theta^T):    g = (Theta^T res)[c]; z0 = y - tau g / p;
//                                   x' = prox(z0); y = x' + beta_k (x' - x_prev)
//   ---- grid barrier ----
// fused: gradient + residual + preconditioner + weighted soft threshold + momentum.
// Vectors live in COMPACTED coordinates (R = nonempty rows, C = nonempty columns);
// every other coordinate has gradient exactly 0 (empty column of Theta), so its
// trajectory is the 1-D recurrence x' = prox(y), y = x' + beta (x' - x_prev): those are
// iterated to completion in registers in one pass (loop interchange; per-coordinate
// arithmetic identical to the reference's).
//
// Precision: WBX_FP32 is the hot path (fp32 values/vectors, FMA); WBX_FP64 reproduces
// the reference arithmetic exactly (sequential in-row sums, no contraction, the
// reference's expression order) and, given the same tau, its iterates BITWISE.
// The step tau is estimated in fp64 accumulation by the reference's power iteration
// (same CounterRng(0x5eed) start vector, 200-iteration cap, 1e-6 relative rule).
#include <cmath>
#include <cooperative_groups.h>

#include "internal.hpp"
#include "sell.cuh"

extern "C" void wbx_set_last_error(const char* msg);

namespace wbx {

namespace {

constexpr int kBlock = 256;
constexpr int kWarpsPerBlock = kBlock / 32;

// output scalars (SolveArgs::out)
enum : int {
    OUT_TAU = 0,
    OUT_TAU_ITERS = 1,
    OUT_ITERS_USED = 2,
    OUT_INITIAL_ENERGY = 3,
    OUT_STATUS = 4,  // 0 ok, 8 nonfinite energy
    OUT_LAMBDA_MAX = 5,
    OUT_COUNT = 8
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
    int have_tau, tau_from_device, max_iters, track, stop_on_ref, decoupled_inline;
    // T-typed state
    void* yC;
    void* xpC;
    void* res;
    void* x0R;
    void* tpC;
    void* thrC;
    // power iteration (fp64)
    double* vC;
    double* wv;
    double* uC;
    double* t64;
    double* part;       // [16][grid] rotating partial sums
    const double* dec_reg;  // [max_iters] decoupled sum w|x_k| (tracking)
    const double* dec_supp; // [max_iters] decoupled support count (tracking)
    double* out;
    double* energies;
    unsigned long long* supports;
    unsigned* bar;
};

__device__ __forceinline__ bool bit_set(const uint32_t* mask, uint64_t i) {
    return (mask[i >> 5] >> (i & 31)) & 1u;
}

__device__ __forceinline__ uint64_t rng_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ull * (i + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double rng_u01(uint64_t v) {
    return (static_cast<double>(v >> 11) + 0.5) * 0x1p-53;
}
// i-th draw of CounterRng(seed).next_normal() (rng.hpp:30-43): pairs (cos, sin).
__device__ __forceinline__ double rng_normal(uint64_t seed, uint64_t i) {
    const uint64_t m = i >> 1;
    const double u1 = rng_u01(rng_at(seed, 2 * m));
    const double u2 = rng_u01(rng_at(seed, 2 * m + 1));
    const double r = sqrt(-2.0 * log(u1));
    const double a = 2.0 * M_PI * u2;
    return (i & 1) ? r * sin(a) : r * cos(a);
}

// ---------------------------------------------------------------- precision traits
template <typename T>
struct Prec;

template <>
struct Prec<float> {
    __device__ static float dot(const SellView& M, uint32_t s, int lane, const float* x) {
        return sell_dot_f32(M, s, lane, x);
    }
    __device__ static double dot_pw(const SellView& M, uint32_t s, int lane, const double* x) {
        return sell_dot_f32v_f64(M, s, lane, x);
    }
    __device__ static float sub(float a, float b) { return a - b; }
    // z0 = y - (tau/p) g   (tp = tau/p precomputed in fp64, rounded once)
    __device__ static float z0(float y, float g, float tp, double, double) { return fmaf(-tp, g, y); }
    __device__ static float prox(float z0, float thr) {
        const float a = fabsf(z0) - thr;
        return a > 0.f ? (z0 > 0.f ? a : -a) : 0.f;
    }
    __device__ static float momentum(float xn, float xp, float beta) {
        return fmaf(beta, xn - xp, xn);
    }
    __device__ static float beta(const SolveArgs& a, int k) { return a.beta32[k - 1]; }
};

template <>
struct Prec<double> {
    __device__ static double dot(const SellView& M, uint32_t s, int lane, const double* x) {
        return sell_dot_f64_exact(M, s, lane, x);
    }
    __device__ static double dot_pw(const SellView& M, uint32_t s, int lane, const double* x) {
        return sell_dot_f64_exact(M, s, lane, x);
    }
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

// ---------------------------------------------------------------- decoupled coordinates
// Coordinates with an empty Theta column: g == 0 exactly, so z0 == y and the iterate
// is prox + momentum only. Runs K iterations per coordinate in registers and stops as
// soon as x' == x_prev == 0 (then y == 0 forever: a fixed point).
// mode 0: write x_K into x_full.  mode 1: per-iteration warp sums of w|x_k| and
// [x_k != 0] into wsum[(k-1) * nwarps + gwarp] (deterministic, no atomics).
template <typename T>
__device__ void decoupled_pass(const SolveArgs& a, double tau, int K, int mode, uint64_t gthread,
                               uint64_t nthreads, double* wreg, double* wsup, uint64_t nwarps) {
    const int lane = threadIdx.x & 31;
    const uint64_t gwarp = gthread >> 5;
    // warp-uniform trip count so warp sums stay well-defined in mode 1
    const uint64_t trips = (a.n + nthreads - 1) / nthreads;
    for (uint64_t t = 0; t < trips; ++t) {
        const uint64_t i = t * nthreads + gthread;
        bool active = i < a.n && !bit_set(a.isC, i);
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
        }
    }
}

// ---------------------------------------------------------------- the persistent kernel
template <typename T>
__global__ void __launch_bounds__(kBlock) solve_kernel(SolveArgs a) {
    __shared__ double red[kWarpsPerBlock + 1];
    const unsigned G = gridDim.x;
    const int lane = threadIdx.x & 31;
    const uint32_t gwarp = (blockIdx.x * kBlock + threadIdx.x) >> 5;
    const uint32_t nwarps = G * kWarpsPerBlock;
    const uint64_t gthread = static_cast<uint64_t>(blockIdx.x) * kBlock + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(G) * kBlock;
    T* yC = static_cast<T*>(a.yC);
    T* xpC = static_cast<T*>(a.xpC);
    T* res = static_cast<T*>(a.res);
    T* x0R = static_cast<T*>(a.x0R);
    T* tpC = static_cast<T*>(a.tpC);
    T* thrC = static_cast<T*>(a.thrC);
    unsigned slot = 0;  // rotating partials slot
    auto part = [&](int which) { return a.part + static_cast<uint64_t>((slot * 4 + which) % 16) * G; };

    // ---- init: compacted copies of x0; warm start x = x_prev = y = x0 (solver.cpp:115-117)
    for (uint64_t c = gthread; c < a.nC; c += nthreads) {
        const T v = static_cast<T>(a.x0_full[a.C_glob[c]]);
        yC[c] = v;
        xpC[c] = v;
    }
    for (uint64_t r = gthread; r < a.nR; r += nthreads) x0R[r] = static_cast<T>(a.x0_full[a.R_glob[r]]);

    // ---- step size: estimate_step (solver.cpp:69-99)
    double tau = a.tau_from_device ? a.out[OUT_TAU] : a.tau_given;
    if (!a.have_tau && !a.tau_from_device) {
        // v = CounterRng(0x5eed) normals over ALL n, normalised by the full norm; only the
        // C part of v ever meets Theta (v is zero outside C after the first product).
        double s2 = 0.0;
        for (uint64_t i = gthread; i < a.n; i += nthreads) {
            const double v = rng_normal(0x5eedull, i);
            s2 += v * v;
        }
        s2 = block_sum<kBlock>(s2, red);
        if (threadIdx.x == 0) part(0)[blockIdx.x] = s2;
        grid_sync(a.bar, G);
        const double nv = sqrt(reduce_partials(part(0), G, red));
        ++slot;
        for (uint64_t c = gthread; c < a.nC; c += nthreads) {
            const double v = rng_normal(0x5eedull, a.C_glob[c]) / nv;
            a.vC[c] = v;
            a.uC[c] = a.ispC[c] * v;
        }
        grid_sync(a.bar, G);
        double lambda_prev = 0.0;
        int it = 0;
        bool zero_op = false;
        for (; it < 200; ++it) {
            // t = Theta (isp .* v)
            for (uint32_t s = gwarp; s < a.A.slices; s += nwarps) {
                const double t = Prec<T>::dot_pw(a.A, s, lane, a.uC);
                const uint32_t r = s * kWarp + lane;
                if (r < a.A.rows) a.t64[r] = t;
            }
            grid_sync(a.bar, G);
            // w = isp .* (Theta^T t); partial <v,w>, <w,w>
            double pl = 0.0, pn = 0.0;
            for (uint32_t s = gwarp; s < a.T.slices; s += nwarps) {
                const double g = Prec<T>::dot_pw(a.T, s, lane, a.t64);
                const uint32_t c = s * kWarp + lane;
                if (c < a.T.rows) {
                    const double w = g * a.ispC[c];
                    a.wv[c] = w;
                    pl += a.vC[c] * w;
                    pn += w * w;
                }
            }
            pl = block_sum<kBlock>(pl, red);
            pn = block_sum<kBlock>(pn, red);
            if (threadIdx.x == 0) {
                part(0)[blockIdx.x] = pl;
                part(1)[blockIdx.x] = pn;
            }
            grid_sync(a.bar, G);
            const double lambda = reduce_partials(part(0), G, red);
            const double nw = sqrt(reduce_partials(part(1), G, red));
            ++slot;
            if (nw == 0.0) {
                zero_op = true;
                ++it;
                break;
            }
            for (uint64_t c = gthread; c < a.nC; c += nthreads) {
                const double v = a.wv[c] / nw;
                a.vC[c] = v;
                a.uC[c] = a.ispC[c] * v;
            }
            if (it > 0 && fabs(lambda - lambda_prev) <= 1e-6 * fabs(lambda)) {
                lambda_prev = lambda;
                ++it;
                break;
            }
            lambda_prev = lambda;
            grid_sync(a.bar, G);
        }
        tau = (zero_op || lambda_prev <= 0.0) ? 1.0 : 1.0 / (lambda_prev * a.step_safety);
        if (gthread == 0) {
            a.out[OUT_TAU_ITERS] = it > 200 ? 200 : it;
            a.out[OUT_LAMBDA_MAX] = lambda_prev;
        }
    }
    if (gthread == 0 && !a.tau_from_device) {
        a.out[OUT_TAU] = tau;
        if (a.have_tau) a.out[OUT_TAU_ITERS] = 0;
    }

    // ---- per-coordinate constants on C: tau/p and tau*lambda*w/p
    for (uint64_t c = gthread; c < a.nC; c += nthreads) {
        tpC[c] = static_cast<T>(tau / a.pC[c]);
        thrC[c] = static_cast<T>(thr_exact(tau, a.lambda, a.wC[c], a.pC[c]));
    }

    // ---- tracking: initial energy E(x0) (solver.cpp:118)
    double stop_gap = 0.0, quad_nonR = 0.0;
    if (a.track) {
        double qn = 0.0, rg = 0.0;
        for (uint64_t i = gthread; i < a.n; i += nthreads) {
            const double x0 = a.x0_full[i];
            if (!bit_set(a.isR, i)) qn += x0 * x0;
            rg += a.w_full[i] * fabs(x0);
        }
        double qr = 0.0;
        for (uint32_t s = gwarp; s < a.A.slices; s += nwarps) {
            const uint32_t r = s * kWarp + lane;
            const double t = static_cast<double>(Prec<T>::dot(a.A, s, lane, yC));
            if (r < a.A.rows) {
                const double d = t - static_cast<double>(x0R[r]);
                qr += d * d;
            }
        }
        qn = block_sum<kBlock>(qn, red);
        rg = block_sum<kBlock>(rg, red);
        qr = block_sum<kBlock>(qr, red);
        if (threadIdx.x == 0) {
            part(0)[blockIdx.x] = qn;
            part(1)[blockIdx.x] = rg;
            part(2)[blockIdx.x] = qr;
        }
        grid_sync(a.bar, G);
        quad_nonR = reduce_partials(part(0), G, red);
        const double reg0 = reduce_partials(part(1), G, red);
        const double quadR0 = reduce_partials(part(2), G, red);
        ++slot;
        const double e0 = 0.5 * (quadR0 + quad_nonR) + a.lambda * reg0;
        stop_gap = a.rel_tol * e0;
        if (gthread == 0) a.out[OUT_INITIAL_ENERGY] = e0;
    }

    // ---- decoupled coordinates (independent of everything else)
    if (a.decoupled_inline) decoupled_pass<T>(a, tau, a.max_iters, 0, gthread, nthreads, nullptr, nullptr, 0);

    grid_sync(a.bar, G);

    // ---- the FISTA / ISTA loop (solver.cpp:121-151)
    int k = 1;
    for (; k <= a.max_iters; ++k) {
        // phase A: res = Theta y - x0 on nonempty rows
        for (uint32_t s = gwarp; s < a.A.slices; s += nwarps) {
            const T acc = Prec<T>::dot(a.A, s, lane, yC);
            const uint32_t r = s * kWarp + lane;
            if (r < a.A.rows) res[r] = Prec<T>::sub(acc, x0R[r]);
        }
        grid_sync(a.bar, G);
        // phase T: gradient on nonempty columns + fused step / prox / momentum
        const T beta = Prec<T>::beta(a, k);
        double reg = 0.0, sup = 0.0;
        for (uint32_t s = gwarp; s < a.T.slices; s += nwarps) {
            const T g = Prec<T>::dot(a.T, s, lane, res);
            const uint32_t c = s * kWarp + lane;
            if (c < a.T.rows) {
                const T y = yC[c], xp = xpC[c];
                const T z0 = Prec<T>::z0(y, g, tpC[c], tau, a.pC[c]);
                const T xn = Prec<T>::prox(z0, thrC[c]);
                yC[c] = Prec<T>::momentum(xn, xp, beta);
                xpC[c] = xn;
                if (a.track) {
                    reg += a.wC[c] * fabs(static_cast<double>(xn));
                    sup += xn != T(0) ? 1.0 : 0.0;
                }
            }
        }
        grid_sync(a.bar, G);
        if (a.track) {
            // energy(x') (solver.cpp:130, :44-55): Theta x' on rows R
            double qr = 0.0;
            for (uint32_t s = gwarp; s < a.A.slices; s += nwarps) {
                const uint32_t r = s * kWarp + lane;
                const double t = static_cast<double>(Prec<T>::dot(a.A, s, lane, xpC));
                if (r < a.A.rows) {
                    const double d = t - static_cast<double>(x0R[r]);
                    qr += d * d;
                }
            }
            qr = block_sum<kBlock>(qr, red);
            reg = block_sum<kBlock>(reg, red);
            sup = block_sum<kBlock>(sup, red);
            if (threadIdx.x == 0) {
                part(0)[blockIdx.x] = qr;
                part(1)[blockIdx.x] = reg;
                part(2)[blockIdx.x] = sup;
            }
            grid_sync(a.bar, G);
            const double quadR = reduce_partials(part(0), G, red);
            const double regC = reduce_partials(part(1), G, red);
            const double supC = reduce_partials(part(2), G, red);
            ++slot;
            const double e = 0.5 * (quadR + quad_nonR) + a.lambda * (regC + a.dec_reg[k - 1]);
            if (gthread == 0) {
                a.energies[k - 1] = e;
                a.supports[k - 1] = static_cast<unsigned long long>(supC + a.dec_supp[k - 1]);
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
    const int used = k - 1 > a.max_iters ? a.max_iters : k - 1;
    if (gthread == 0) a.out[OUT_ITERS_USED] = used;
    // ---- x_final on C back into the full coefficient vector
    for (uint64_t c = gthread; c < a.nC; c += nthreads) a.x_full[a.C_glob[c]] = static_cast<double>(xpC[c]);
}

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

// wreg/wsup [K][nwarps] -> dec_reg/dec_supp [K], fixed order
__global__ void reduce_rows_kernel(const double* w, uint64_t nwarps, int K, double* outp) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    double s = 0.0;
    for (uint64_t j = 0; j < nwarps; ++j) s += w[static_cast<uint64_t>(k) * nwarps + j];
    outp[k] = s;
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
    wbx::DevBuf<double> pC, wC, ispC, w_full, p_full, beta64;
    wbx::DevBuf<float> beta32;
    wbx::DevBuf<unsigned char> state;  // yC, xpC, res, x0R, tpC, thrC (T-typed)
    wbx::DevBuf<double> vC, wv, uC, t64, part, out, energies, dec_reg, dec_supp, wreg, wsup;
    wbx::DevBuf<unsigned long long> supports;
    wbx::DevBuf<unsigned> bar;
    wbx::DevBuf<double> u0, x0full, xfull, uout;
    int grid = 0;
    int dec_grid = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    uint64_t last_launches = 0;
    float last_solve_ms = 0.f;
};

namespace wbx {

namespace {

template <typename T>
int occupancy_grid(wbx_ctx* ctx) {
    int per_sm = 0;
    WBX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_kernel<T>, kBlock, 0));
    if (per_sm < 1) fail(WBX_CUDA_ERROR, "solver kernel cannot be resident");
    return per_sm * ctx->num_sms;
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
    a.have_tau = s->cfg.tau > 0.0;
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
    a.yC = carve(nC);
    a.xpC = carve(nC);
    a.res = carve(nR);
    a.x0R = carve(nR);
    a.tpC = carve(nC);
    a.thrC = carve(nC);
    a.vC = s->vC.p;
    a.wv = s->wv.p;
    a.uC = s->uC.p;
    a.t64 = s->t64.p;
    a.part = s->part.p;
    a.dec_reg = s->dec_reg.p;
    a.dec_supp = s->dec_supp.p;
    a.out = s->out.p;
    a.energies = s->energies.p;
    a.supports = s->supports.p;
    a.bar = s->bar.p;
    return a;
}

template <typename T>
void run_solve(wbx_solver* s, const double* x0_full, double* x_full, cudaStream_t st) {
    SolveArgs a = make_args<T>(s, x0_full, x_full);
    wbx_ctx* ctx = s->ctx;
    WBX_CUDA(cudaMemsetAsync(s->out.p, 0, s->out.bytes(), st));
    void* params[] = {&a};
    if (!a.track) {
        WBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(solve_kernel<T>), dim3(s->grid),
                                             dim3(kBlock), params, 0, st));
        count_launch(ctx);
        return;
    }
    // Tracking (energies / supports / ref_energy stopping rule, solver.cpp:130-150):
    // (1) tau-only pass; (2) decoupled per-iteration sums with that tau; (3) reduce them;
    // (4) tracked solve; (5) decoupled final write at the iteration count used.
    SolveArgs pre = a;
    pre.max_iters = 0;
    pre.track = 0;
    pre.decoupled_inline = 0;
    pre.stop_on_ref = 0;
    void* pparams[] = {&pre};
    WBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(solve_kernel<T>), dim3(s->grid),
                                         dim3(kBlock), pparams, 0, st));
    const uint64_t nthreads = static_cast<uint64_t>(s->dec_grid) * kBlock;
    const uint64_t nwarps = nthreads / 32;
    const int K = a.max_iters;
    if (K > 0) {
        WBX_CUDA(cudaMemsetAsync(s->wreg.p, 0, s->wreg.bytes(), st));
        WBX_CUDA(cudaMemsetAsync(s->wsup.p, 0, s->wsup.bytes(), st));
        decoupled_kernel<T><<<s->dec_grid, kBlock, 0, st>>>(a, 1, s->wreg.p, s->wsup.p, s->out.p);
        reduce_rows_kernel<<<(K + 127) / 128, 128, 0, st>>>(s->wreg.p, nwarps, K, s->dec_reg.p);
        reduce_rows_kernel<<<(K + 127) / 128, 128, 0, st>>>(s->wsup.p, nwarps, K, s->dec_supp.p);
        count_launch(ctx, 3);
    }
    a.tau_from_device = 1;
    WBX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(solve_kernel<T>), dim3(s->grid),
                                         dim3(kBlock), params, 0, st));
    decoupled_kernel<T><<<s->dec_grid, kBlock, 0, st>>>(a, 0, nullptr, nullptr, s->out.p);
    count_launch(ctx, 3);
    WBX_CUDA(cudaGetLastError());
}

template <typename T>
void alloc_state(wbx_solver* s) {
    const wbx_op* op = s->op;
    auto rnd = [](uint64_t count) { return ((count * sizeof(T) + 255) / 256) * 256; };
    s->state.alloc(4 * rnd(op->nC) + 2 * rnd(op->nR) + 256);
}

}  // namespace

void solver_setup(wbx_solver* s, const double* p, const double* w) {
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
    s->p_full.alloc(n);
    s->p_full.upload(p, n, st);
    s->w_full.alloc(n);
    s->w_full.upload(w, n, st);
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
    if (s->cfg.precision == WBX_FP64) {
        alloc_state<double>(s);
        s->grid = occupancy_grid<double>(s->ctx);
    } else {
        alloc_state<float>(s);
        s->grid = occupancy_grid<float>(s->ctx);
    }
    s->dec_grid = 4 * s->ctx->num_sms;
    s->vC.alloc(nC ? nC : 1);
    s->wv.alloc(nC ? nC : 1);
    s->uC.alloc(nC ? nC : 1);
    s->t64.alloc(op->nR ? op->nR : 1);
    s->part.alloc(16 * static_cast<uint64_t>(s->grid));
    s->out.alloc(OUT_COUNT);
    s->bar.alloc(2);
    WBX_CUDA(cudaMemsetAsync(s->bar.p, 0, s->bar.bytes(), st));
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
    WBX_CUDA(cudaEventCreate(&s->ev0));
    WBX_CUDA(cudaEventCreate(&s->ev1));
    WBX_CUDA(cudaStreamSynchronize(st));
}

void solver_run(wbx_solver* s, const double* x0_full_dev, double* x_full_dev) {
    cudaStream_t st = s->ctx->stream;
    WBX_CUDA(cudaEventRecord(s->ev0, st));
    if (s->cfg.precision == WBX_FP64)
        run_solve<double>(s, x0_full_dev, x_full_dev, st);
    else
        run_solve<float>(s, x0_full_dev, x_full_dev, st);
    WBX_CUDA(cudaEventRecord(s->ev1, st));
}

void solver_report(wbx_solver* s, wbx_report* rep) {
    cudaStream_t st = s->ctx->stream;
    double out[OUT_COUNT];
    WBX_CUDA(cudaMemcpyAsync(out, s->out.p, sizeof out, cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    WBX_CUDA(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
    s->last_solve_ms = ms;
    if (out[OUT_STATUS] == 8.0) fail(WBX_NONFINITE_ENERGY, "solver diverged (non-finite energy)");
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

}  // namespace wbx

namespace wbx {

wbx_solver* solver_new(wbx_ctx* ctx, const wbx_op* op, wbx_basis* basis, double lambda,
                       const wbx_solver_cfg& cfg, int accelerate) {
    if (cfg.precision != WBX_FP32 && cfg.precision != WBX_FP64)
        fail(WBX_BAD_SPEC, "precision must be 32 or 64");
    if (cfg.max_iters > 0x7fffffffull) fail(WBX_TOO_LARGE, "max_iters too large");
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
    delete s;
}

void solver_alloc_images(wbx_solver* s) {
    s->u0.alloc(s->n);
    s->x0full.alloc(s->n);
    s->xfull.alloc(s->n);
    s->uout.alloc(s->n);
}

}  // namespace wbx

extern "C" {

int wbx_deblur_dev(wbx_solver* s, const double* u0_dev, double* u_dev, int clamp) {
    try {
        if (!s || !u0_dev || !u_dev) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_deblur_dev");
        cudaStream_t st = s->ctx->stream;
        const uint64_t before = s->ctx->launches;
        wbx::analyze_dev(s->basis, u0_dev, s->x0full.p, st);
        wbx::solver_run(s, s->x0full.p, s->xfull.p);
        wbx::synthesize_dev(s->basis, s->xfull.p, u_dev, st);
        if (clamp) wbx::launch_clamp(s->ctx, u_dev, s->n, st);
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
        WBX_CUDA(cudaMemcpyAsync(s->u0.p, u0, s->n * sizeof(double), cudaMemcpyHostToDevice, st));
        const int rc = wbx_deblur_dev(s, s->u0.p, s->uout.p, clamp);
        if (rc != WBX_OK) return rc;
        WBX_CUDA(cudaMemcpyAsync(u, s->uout.p, s->n * sizeof(double), cudaMemcpyDeviceToHost, st));
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
        if (cudaEventElapsedTime(&ms, s->ev0, s->ev1) != cudaSuccess) return WBX_CUDA_ERROR;
        *solve_ms = ms;
    }
    return WBX_OK;
}

}  // extern "C"
