// Step estimate (`estimate_step`, proj/src/solver.cpp:69-99) for translation-invariant
// operators, computed block-diagonally in the Fourier domain of the translation group.
//
// The reference's estimate is the power iteration on M = P^-1/2 Theta^T Theta P^-1/2 from
// v0 = CounterRng(0x5eed) normals over all n (normalised): lambda_it = <v_it, M v_it> with
// v_it = M^it v0 / |M^it v0|, stopping at the first it > 0 with |lambda_it - lambda_it-1| <=
// 1e-6 lambda_it (cap 200), tau = 1 / (lambda * step_safety). With the moments
// mu_p = v0^T M^p v0, lambda_0 = mu_1 / |v0|^2 and lambda_it = mu_{2it+1} / mu_{2it}.
//
// A stationary Theta_K (the reference's threshold keeps whole circulant generator groups,
// theta.cpp:206-276) commutes with the image translations by 2^J pixels: the group
// Z_g0 x Z_g1, g = dims / 2^J, moves a coefficient of a level-j band by 2^(J-j) positions.
// A band position p splits into an orbit representative a = p mod s and a group element
// h = p div s (s = band shape / g), and Theta[(o', h'), (o, h)] depends only on h' - h. The
// group's Fourier transform therefore block-diagonalises Theta into one small matrix per
// frequency f, Theta^_f[o', o] = sum over the row (o', 0) of Theta of val * e^{+2 pi i f.h / g}
// (nRo x nCo: the row / column orbits that hold nonzeros; 38 x 12 at C1/C2), and
//     mu_p = (1 / NG) sum_f  v^_f^H  M^_f^p  v^_f,   M^_f = D Theta^_f^H Theta^_f D,
// D = P^-1/2 per column orbit, v^_f the transform of v0 on the column orbits (e^{-}).
// So the reference's power iteration is NG independent power iterations on nCo x nCo
// matrices (4096 of 12 x 12 at C2), run to the cap in fp64 and summed per moment: the
// reference's lambda sequence, stopping index and tau, to fp64 rounding (1e-15 on the golden
// operators vs 2e-8 for the fp32 Lanczos estimate), without touching the full operator.
//
// Applicability (checked exactly once per operator and layout, host, O(n + nnz)): every row
// of Theta equals its orbit representative's row shifted by its group element (entry sets and
// values bitwise); P constant on every column orbit (checked per solver, 1e-12 relative, the
// representative's value is used); nCo <= 16, g0, g1 <= 1024. Otherwise (spatially varying
// operators, a top-K boundary that splits a generator group) the solver keeps the Lanczos /
// power-iteration estimate.
//
// f and -f carry conjugate blocks and transforms (Theta and v0 are real), hence equal
// moments: only the half spectrum is evaluated (2050 of 4096 frequencies at C2).
//
// Device work per estimate (7 launches, all image-independent, in the step-estimate graph):
//   circ_gram_kernel     (forked stream) G_f = Theta^_f^H Theta^_f per frequency from the
//                        representative rows staged in shared memory: lanes over (row, orbit) pairs
//                        for Theta^_f, then over (i, j) for G_f (also the spectral FISTA's blocks)
//   circ_norm_kernel     |v0|^2 over all n (one log per Box-Muller pair; block partials)
//   circ_dft1/0_kernel   v^ on the column orbits (separable DFT, twiddle tables)
//   circ_lanczos_kernel  half a warp per frequency: M^_f = D G_f D; Lanczos with full
//                        reorthogonalisation -> the real tridiagonal T_f (<= nCo steps, exact:
//                        the Krylov space is the block's)
//   circ_power_kernel    one thread per frequency: the 201 power steps on T_f (5 fma per row
//                        instead of a dense complex matvec), exact power-of-two rescaling, the
//                        402 moments
//   circ_reduce_kernel   per moment, the sum over frequencies with a common exponent (fixed
//                        order); its last block evaluates lambda_it for every it in parallel, the
//                        reference's stopping rule and tau (circ_final_body)
#include <cmath>
#include <cstring>
#include <string>

#include "internal.hpp"
#include "rng.cuh"
#include "wbx_diag.h"

#ifndef WBX_CIRC_PROF
#define WBX_CIRC_PROF 0
#endif

extern "C" void wbx_set_last_error(const char* msg);

namespace wbx {

namespace {

constexpr int kCircMaxCo = 16;      // column orbits (two lanes per row of M^_f)
constexpr int kCircMoments = 402;   // mu_0 .. mu_401 (lambda_199 needs mu_399, the sentinel mu_400)
constexpr int kCircWarps = 2;       // warps per block of circ_lanczos_kernel (two frequencies each)
constexpr int kCircNormBlocks = 296;

struct CircOrbit {  // a column orbit: flat index of (h0, h1) = off + (a0 + s0 h0) * W + a1 + s1 h1
    uint32_t off, W, a0, a1, s0, s1;
};

}  // namespace

struct CircPlan {
    bool ok = false;
    std::string why;
    uint32_t g0 = 1, g1 = 1, NG = 1, nRo = 0, nCo = 0;
    uint64_t n = 0;
    std::vector<uint32_t> c_rep;  // column orbit -> flat index of its representative (h = 0)
    std::vector<CircOrbit> h_orb;
    std::vector<uint32_t> h_eoff, h_eh;
    std::vector<double> h_eval;
    std::vector<double2> h_tw0, h_tw1;
    std::vector<uint32_t> h_fhalf;  // half spectrum: f << 1 | (weight 2)
    std::vector<int> h_hidx;        // frequency -> half-spectrum index, or -1 - its conjugate's
    std::vector<CircOrbit> h_rorb;  // row orbits, in the order of the representative rows
    bool fista_ok = false;          // the spectral FISTA engine applies (circ_fista_kernel)
    std::string fista_why;
    bool uploaded = false;
    DevBuf<uint32_t> fhalf;
    DevBuf<int> hidx;
    DevBuf<CircOrbit> rorb;
    DevBuf<CircOrbit> orb;
    DevBuf<uint32_t> eoff;  // [nRo * nCo + 1]: entries of representative row r, column orbit j
    DevBuf<uint32_t> eh;    // h0 << 16 | h1
    DevBuf<double> eval;
    DevBuf<double2> tw0, tw1;  // e^{2 pi i k / g}
};

namespace {

// ----------------------------------------------------------------------------- device

// |v0|^2 over all n. The Box-Muller pair (2m, 2m+1) has v_2m^2 + v_2m+1^2 = r_m^2 = -2 log u1_m,
// so the sum needs one log per pair (an odd n's last draw is squared directly). Block b sums
// its contiguous chunk of pairs, threads strided, fixed tree.
__global__ void circ_norm_kernel(uint64_t n, double* part) {
    __shared__ double red[256];
    const uint64_t pairs = n / 2;
    const uint64_t chunk = (pairs + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = chunk * blockIdx.x, hi = lo + chunk < pairs ? lo + chunk : pairs;
    double s = 0.0;
    for (uint64_t m = lo + threadIdx.x; m < hi; m += blockDim.x) s += -2.0 * log(rng_u01(rng_at(0x5eedull, 2 * m)));
    if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        const double v = rng_normal(0x5eedull, n - 1);
        s += v * v;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// DFT along h1 of v0 on column orbit blockIdx.y, row h0 = blockIdx.x: t1[oc][h0][f1]
__global__ void circ_dft1_kernel(const CircOrbit* orb, uint32_t g0, uint32_t g1, const double2* tw1, double2* t1) {
    extern __shared__ double2 circ_smem[];
    double* sv = reinterpret_cast<double*>(circ_smem);
    const uint32_t oc = blockIdx.y, h0 = blockIdx.x;
    const CircOrbit o = orb[oc];
    for (uint32_t j = threadIdx.x; j < g1; j += blockDim.x) {
        const uint64_t flat = static_cast<uint64_t>(o.off) + static_cast<uint64_t>(o.a0 + o.s0 * h0) * o.W + o.a1 + o.s1 * j;
        sv[j] = rng_normal(0x5eedull, flat);
    }
    __syncthreads();
    for (uint32_t f1 = threadIdx.x; f1 < g1; f1 += blockDim.x) {
        double re = 0.0, im = 0.0;
        uint32_t k = 0;  // f1 * j mod g1
        for (uint32_t j = 0; j < g1; ++j) {
            const double2 w = tw1[k];
            re = fma(sv[j], w.x, re);
            im = fma(-sv[j], w.y, im);
            k += f1;
            if (k >= g1) k -= g1;
        }
        t1[(static_cast<uint64_t>(oc) * g0 + h0) * g1 + f1] = make_double2(re, im);
    }
}

// DFT along h0: vh[f0 * g1 + f1][oc]
__global__ void circ_dft0_kernel(uint32_t nCo, uint32_t g0, uint32_t g1, const double2* tw0, const double2* t1,
                                 double2* vh) {
    extern __shared__ double2 circ_smem[];
    double2* st = circ_smem;
    const uint32_t oc = blockIdx.y, f1 = blockIdx.x;
    for (uint32_t h0 = threadIdx.x; h0 < g0; h0 += blockDim.x)
        st[h0] = t1[(static_cast<uint64_t>(oc) * g0 + h0) * g1 + f1];
    __syncthreads();
    for (uint32_t f0 = threadIdx.x; f0 < g0; f0 += blockDim.x) {
        double re = 0.0, im = 0.0;
        uint32_t k = 0;
        for (uint32_t h0 = 0; h0 < g0; ++h0) {
            const double2 w = tw0[k], x = st[h0];  // x * conj(w)
            re = fma(x.x, w.x, fma(x.y, w.y, re));
            im = fma(x.y, w.x, fma(-x.x, w.y, im));
            k += f0;
            if (k >= g0) k -= g0;
        }
        vh[(static_cast<uint64_t>(f0) * g1 + f1) * nCo + oc] = make_double2(re, im);
    }
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// Half a warp per frequency of the half spectrum, two frequencies per warp (lane i < nCo of a
// half owns column orbit i): Theta^_f row by row from the representative rows (staged in shared
// memory once per block), G_f = Theta^_f^H Theta^_f (lane i: row i), written to gram[hf] as
// nCo x nCo complex fp64. G_f is the Fourier block of Theta^T Theta: the step estimate scales it
// by D = P^-1/2, the spectral FISTA engine applies it as is.
// Copy n complex values src(i) -> dst(i) with every load of a thread issued before its stores
// (one memory round trip per call, not one per element)
template <typename Src, typename Dst>
__device__ __forceinline__ void batched_copy(uint32_t n, Src src, Dst dst) {
    constexpr int kB = 8;
    for (uint32_t base = 0; base < n; base += kB * blockDim.x) {
        double2 v[kB];
#pragma unroll
        for (int r = 0; r < kB; ++r) {
            const uint32_t i = base + r * blockDim.x + threadIdx.x;
            if (i < n) v[r] = src(i);
        }
#pragma unroll
        for (int r = 0; r < kB; ++r) {
            const uint32_t i = base + r * blockDim.x + threadIdx.x;
            if (i < n) dst(i, v[r]);
        }
    }
}

constexpr int kGramWarps = 4;  // frequencies per block of circ_gram_kernel

__global__ void __launch_bounds__(kGramWarps * 32) circ_gram_kernel(
    uint32_t nhalf, const uint32_t* __restrict__ fhalf, uint32_t g1, uint32_t g0, uint32_t nRo, uint32_t nCo,
    const uint32_t* __restrict__ eoff, const uint32_t* __restrict__ eh, const double* __restrict__ eval,
    const double2* __restrict__ tw0, const double2* __restrict__ tw1, double2* __restrict__ gram, uint32_t nent) {
    // the representative rows and twiddles, staged once per block (loads issued before the stores)
    extern __shared__ double2 circ_smem[];
    const uint32_t nTh = nRo * nCo;  // Theta^_f entries of one frequency
    double2* s_th = circ_smem;                                 // [kGramWarps][nRo][nCo]
    double2* s_tw0 = s_th + kGramWarps * nTh;
    double2* s_tw1 = s_tw0 + g0;
    double* s_val = reinterpret_cast<double*>(s_tw1 + g1);
    uint32_t* s_eh = reinterpret_cast<uint32_t*>(s_val + nent);
    uint32_t* s_eoff = s_eh + nent;
    batched_copy(g0, [&](uint32_t i) { return tw0[i]; }, [&](uint32_t i, double2 v) { s_tw0[i] = v; });
    batched_copy(g1, [&](uint32_t i) { return tw1[i]; }, [&](uint32_t i, double2 v) { s_tw1[i] = v; });
    batched_copy(
        nent, [&](uint32_t i) { return make_double2(eval[i], __longlong_as_double(static_cast<long long>(eh[i]))); },
        [&](uint32_t i, double2 v) {
            s_val[i] = v.x;
            s_eh[i] = static_cast<uint32_t>(__double_as_longlong(v.y));
        });
    batched_copy(
        nTh + 1, [&](uint32_t i) { return make_double2(__longlong_as_double(static_cast<long long>(eoff[i])), 0.0); },
        [&](uint32_t i, double2 v) { s_eoff[i] = static_cast<uint32_t>(__double_as_longlong(v.x)); });
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t hf = blockIdx.x * kGramWarps + w;
    if (hf >= nhalf) return;  // whole warp
    const uint32_t f = fhalf[hf] >> 1;
    const uint32_t f0 = f / g1, f1 = f % g1;
    const uint32_t m0 = (g0 & (g0 - 1)) == 0 ? g0 - 1 : 0, m1 = (g1 & (g1 - 1)) == 0 ? g1 - 1 : 0;
    double2* th = s_th + w * nTh;
    // Theta^_f[r][j] = sum over the entries (j, h) of representative row r of val e^{+2 pi i f.h/g}:
    // every (r, j) pair independently (lanes over pairs)
    for (uint32_t p = lane; p < nTh; p += 32) {
        double re = 0.0, im = 0.0;
        for (uint32_t e = s_eoff[p]; e < s_eoff[p + 1]; ++e) {
            const uint32_t h = s_eh[e];
            const uint32_t a0 = f0 * (h >> 16), a1 = f1 * (h & 0xffffu);
            const double2 ph = cmul(s_tw0[m0 ? (a0 & m0) : a0 % g0], s_tw1[m1 ? (a1 & m1) : a1 % g1]);
            re = fma(s_val[e], ph.x, re);
            im = fma(s_val[e], ph.y, im);
        }
        th[p] = make_double2(re, im);
    }
    __syncwarp();
    // G_f[i][j] = sum_r conj(Theta^[r][i]) Theta^[r][j]: every (i, j) independently, two chains
    double2* G = gram + static_cast<uint64_t>(hf) * nCo * nCo;
    for (uint32_t p = lane; p < nCo * nCo; p += 32) {
        const uint32_t i = p / nCo, j = p % nCo;
        double r0 = 0.0, i0 = 0.0, r1 = 0.0, i1 = 0.0;
        uint32_t r = 0;
        for (; r + 1 < nRo; r += 2) {
            const double2 a = th[r * nCo + i], b = th[r * nCo + j];
            const double2 c = th[(r + 1) * nCo + i], d = th[(r + 1) * nCo + j];
            r0 = fma(a.x, b.x, fma(a.y, b.y, r0));
            i0 = fma(a.x, b.y, fma(-a.y, b.x, i0));
            r1 = fma(c.x, d.x, fma(c.y, d.y, r1));
            i1 = fma(c.x, d.y, fma(-c.y, d.x, i1));
        }
        if (r < nRo) {
            const double2 a = th[r * nCo + i], b = th[r * nCo + j];
            r0 = fma(a.x, b.x, fma(a.y, b.y, r0));
            i0 = fma(a.x, b.y, fma(-a.y, b.x, i0));
        }
        G[p] = make_double2(r0 + r1, i0 + i1);
    }
}


// Half a warp per frequency of the half spectrum (f and -f have conjugate blocks and
// transforms, so equal moments: weight 2; self-conjugate frequencies weight 1), two
// frequencies per warp. Lane i < nCo of a half owns row / component i. Every frequency's
// control flow is the same (the representative rows do not depend on f), so the halves do
// not diverge except at a Lanczos breakdown (per-half flags).
//   1. M^_f = D G_f D from circ_gram_kernel's G_f (lane i: row i), D = P^-1/2 per column orbit
//   2. Lanczos on M^_f from v^_f with full reorthogonalisation (classical Gram-Schmidt, twice):
//      the real tridiagonal T_f (k <= nCo) with v^H M^p v = |v|^2 e1^T T^p e1 for every p;
//      written as {alpha[16], beta[16], |v|^2 (weight folded in), k}
__global__ void __launch_bounds__(kCircWarps * 32) circ_lanczos_kernel(
    uint32_t nhalf, const uint32_t* __restrict__ fhalf, uint32_t nCo, const double2* __restrict__ gram,
    const double* __restrict__ isp, const double2* __restrict__ vh, double* __restrict__ tri) {
    constexpr int kSlots = 2 * kCircWarps;
    __shared__ double2 Ms[kSlots][kCircMaxCo][kCircMaxCo + 1];
    __shared__ double2 Qs[kSlots][kCircMaxCo][kCircMaxCo];
    __shared__ double2 vec[kSlots][kCircMaxCo];  // Theta^ row / current r / q broadcast
    __shared__ double2 cof[kSlots][kCircMaxCo];  // reorthogonalisation coefficients
    const int lane = threadIdx.x & 31, li = lane & 15;
    const int slot = (threadIdx.x >> 5) * 2 + (lane >> 4);
    const uint32_t hf = blockIdx.x * kSlots + slot;
    const uint32_t warp_first = blockIdx.x * kSlots + (threadIdx.x >> 5) * 2;
    if (warp_first >= nhalf) return;  // whole warp
    const bool live = hf < nhalf;
    const uint32_t fw = live ? fhalf[hf] : 0u;
    const uint32_t f = fw >> 1;  // frequency index f0 * g1 + f1; bit 0: weight 2
    const int nc = static_cast<int>(nCo);
    const bool own = li < nc;
    auto half_sum = [](double v) {  // sum over the 16 lanes of this half (identical in every lane)
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };

    // 1. M^_f = D G_f D
    double fro = 0.0;
    if (own) {
        const double di = isp[li];
        const double2* G = gram + static_cast<uint64_t>(live ? hf : 0) * nCo * nCo + static_cast<uint64_t>(li) * nCo;
        for (int j = 0; j < nc; ++j) {
            const double s = di * isp[j];
            const double2 g = G[j];
            const double2 m = make_double2(g.x * s, g.y * s);
            Ms[slot][li][j] = m;
            fro = fma(m.x, m.x, fma(m.y, m.y, fro));
        }
    }
    fro = sqrt(half_sum(fro));

    // 2. Lanczos
    const double2 v = (own && live) ? vh[static_cast<uint64_t>(f) * nCo + li] : make_double2(0.0, 0.0);
    const double vn2 = half_sum(fma(v.x, v.x, v.y * v.y));
    const double rn = vn2 > 0.0 ? 1.0 / sqrt(vn2) : 0.0;
    double2 q = make_double2(v.x * rn, v.y * rn), qprev = make_double2(0.0, 0.0);
    double beta = 0.0;
    int k = 0;
    bool done = !(vn2 > 0.0);
    double al_mine = 0.0, be_mine = 0.0;  // lane li keeps alpha_li and beta_li (T[li-1][li])
    for (int j = 0; j < nc; ++j) {
        __syncwarp();
        if (own) {
            Qs[slot][j][li] = q;
            vec[slot][li] = q;
        }
        __syncwarp();
        double2 y = make_double2(0.0, 0.0);
        if (own) {  // two accumulator chains (even / odd l)
            double2 y1 = make_double2(0.0, 0.0);
#pragma unroll
            for (int l = 0; l < kCircMaxCo; l += 2) {
                if (l < nc) {
                    const double2 m = Ms[slot][li][l], x = vec[slot][l];
                    y.x = fma(m.x, x.x, fma(-m.y, x.y, y.x));
                    y.y = fma(m.x, x.y, fma(m.y, x.x, y.y));
                }
                if (l + 1 < nc) {
                    const double2 m = Ms[slot][li][l + 1], x = vec[slot][l + 1];
                    y1.x = fma(m.x, x.x, fma(-m.y, x.y, y1.x));
                    y1.y = fma(m.x, x.y, fma(m.y, x.x, y1.y));
                }
            }
            y.x += y1.x;
            y.y += y1.y;
        }
        const double alpha = half_sum(own ? fma(q.x, y.x, q.y * y.y) : 0.0);
        double2 r = make_double2(y.x - alpha * q.x - beta * qprev.x, y.y - alpha * q.y - beta * qprev.y);
        for (int pass = 0; pass < 2; ++pass) {  // r -= Q (Q^H r)
            __syncwarp();
            if (own) vec[slot][li] = r;
            __syncwarp();
            if (li <= j) {
                double2 c = make_double2(0.0, 0.0), c1 = make_double2(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < kCircMaxCo; i += 2) {
                    if (i < nc) {
                        const double2 a = Qs[slot][li][i], b = vec[slot][i];  // conj(a) b
                        c.x = fma(a.x, b.x, fma(a.y, b.y, c.x));
                        c.y = fma(a.x, b.y, fma(-a.y, b.x, c.y));
                    }
                    if (i + 1 < nc) {
                        const double2 a = Qs[slot][li][i + 1], b = vec[slot][i + 1];
                        c1.x = fma(a.x, b.x, fma(a.y, b.y, c1.x));
                        c1.y = fma(a.x, b.y, fma(-a.y, b.x, c1.y));
                    }
                }
                cof[slot][li] = make_double2(c.x + c1.x, c.y + c1.y);
            }
            __syncwarp();
            if (own)
                for (int l = 0; l <= j; ++l) {
                    const double2 c = cof[slot][l], a = Qs[slot][l][li];
                    r.x -= fma(c.x, a.x, -c.y * a.y);
                    r.y -= fma(c.x, a.y, c.y * a.x);
                }
        }
        const double bn = sqrt(half_sum(own ? fma(r.x, r.x, r.y * r.y) : 0.0));
        if (!done) {
            if (li == j) al_mine = alpha;
            k = j + 1;
            // full dimension, or an invariant subspace (the Krylov space of v is complete)
            if (j + 1 == nc || !(bn > 1e-13 * fro)) {
                done = true;
            } else {
                if (li == j + 1) be_mine = bn;
                const double rb = 1.0 / bn;
                qprev = q;
                q = make_double2(r.x * rb, r.y * rb);
                beta = bn;
            }
        }
    }
    if (live) {  // tri[hf] = {alpha[16], beta[16], |v|^2 2^(weight bit), k}
        double* t = tri + static_cast<uint64_t>(hf) * (2 * kCircMaxCo + 2);
        t[li] = al_mine;
        t[kCircMaxCo + li] = be_mine;
        if (li == 0) {
            t[2 * kCircMaxCo] = (fw & 1u) ? 2.0 * vn2 : vn2;  // exact
            t[2 * kCircMaxCo + 1] = static_cast<double>(vn2 > 0.0 ? k : 0);
        }
    }
}

// One thread per frequency: 201 power steps y <- T_f y from e1 (K = T's padded size), moments
// mu_2s = |v|^2 |y_s|^2, mu_2s+1 = |v|^2 <y_s, T y_s> as mantissa / exponent [moment][frequency]
// (|y_s+1|^2 = |T y_s|^2 is the next step's even moment); exact power-of-two rescaling every
// 4 steps keeps |y| ~ 1.
template <int K>
__global__ void __launch_bounds__(32) circ_power_kernel(uint32_t nhalf, const double* __restrict__ tri,
                                                        double* __restrict__ mom_m, int* __restrict__ mom_e) {
    const uint32_t hf = blockIdx.x * blockDim.x + threadIdx.x;
    if (hf >= nhalf) return;
    const double* t = tri + static_cast<uint64_t>(hf) * (2 * kCircMaxCo + 2);
    const int k = static_cast<int>(t[2 * kCircMaxCo + 1]);
    double al[K], be[K + 1], y[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        al[i] = i < k ? t[i] : 0.0;
        be[i] = (i > 0 && i < k) ? t[kCircMaxCo + i] : 0.0;
        y[i] = i == 0 ? 1.0 : 0.0;
    }
    be[K] = 0.0;
    int ve;
    const double vm = k > 0 ? frexp(t[2 * kCircMaxCo], &ve) : (ve = 0, 0.0);
    int E = ve;
    double a2 = 1.0;  // |y_0|^2
    auto step = [&](int s, bool rescale) {
        double z[K];
#pragma unroll
        for (int i = 0; i < K; ++i)
            z[i] = fma(al[i], y[i], fma(be[i], i > 0 ? y[i - 1] : 0.0, be[i + 1] * (i + 1 < K ? y[i + 1] : 0.0)));
        double d1[4] = {0, 0, 0, 0}, n2[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < K; ++i) {
            d1[i & 3] = fma(y[i], z[i], d1[i & 3]);
            n2[i & 3] = fma(z[i], z[i], n2[i & 3]);
        }
        const double a1 = (d1[0] + d1[1]) + (d1[2] + d1[3]);
        const double zz = (n2[0] + n2[1]) + (n2[2] + n2[3]);
        mom_m[static_cast<uint64_t>(2 * s) * nhalf + hf] = vm * a2;
        mom_e[static_cast<uint64_t>(2 * s) * nhalf + hf] = E;
        mom_m[static_cast<uint64_t>(2 * s + 1) * nhalf + hf] = vm * a1;
        mom_e[static_cast<uint64_t>(2 * s + 1) * nhalf + hf] = E;
        if (rescale && zz > 0.0 && isfinite(zz)) {
            const int sh = ilogb(zz) / 2;
            const double sc = scalbn(1.0, -sh);  // exact power of two
#pragma unroll
            for (int i = 0; i < K; ++i) y[i] = z[i] * sc;
            a2 = zz * (sc * sc);
            E += 2 * sh;
        } else {
#pragma unroll
            for (int i = 0; i < K; ++i) y[i] = z[i];
            a2 = zz;
        }
    };
    for (int s = 0; s < 200; s += 4) {
        step(s, false);
        step(s + 1, false);
        step(s + 2, false);
        step(s + 3, true);
    }
    step(200, false);
}

// Moment p summed over the half spectrum (fixed order): common exponent X = max(e + ilogb(m)),
// S = sum of m 2^(e - X); block p, threads strided over the frequencies, fixed tree.
__device__ void circ_final_body(uint32_t NG, const double* Sg, const int* Xg, const double* norm_part,
                                int norm_blocks, double step_safety, double* out);

// (the last block to finish then evaluates the lambda sequence: circ_final_body)
__global__ void __launch_bounds__(256) circ_reduce_kernel(uint32_t nhalf, const double* __restrict__ mom_m,
                                                          const int* __restrict__ mom_e, double* S, int* X,
                                                          unsigned* done, uint32_t NG, const double* norm_part,
                                                          int norm_blocks, double step_safety, double* out) {
    __shared__ double rs[256];
    __shared__ int rx[256];
    const int p = blockIdx.x, t = threadIdx.x;
    const double* mm = mom_m + static_cast<uint64_t>(p) * nhalf;
    const int* me = mom_e + static_cast<uint64_t>(p) * nhalf;
    int x = INT_MIN;
    for (uint32_t i = t; i < nhalf; i += 256)
        if (mm[i] != 0.0) x = max(x, me[i] + ilogb(mm[i]));
    rx[t] = x;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (t < k) rx[t] = max(rx[t], rx[t + k]);
        __syncthreads();
    }
    x = rx[0];
    double s = 0.0;
    if (x != INT_MIN)
        for (uint32_t i = t; i < nhalf; i += 256)
            if (mm[i] != 0.0) s += scalbn(mm[i], me[i] - x);
    rs[t] = s;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (t < k) rs[t] += rs[t + k];
        __syncthreads();
    }
    __shared__ bool last;
    if (t == 0) {
        S[p] = rs[0];
        X[p] = x == INT_MIN ? 0 : x;
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    circ_final_body(NG, S, X, norm_part, norm_blocks, step_safety, out);
    if (t == 0) *done = 0;  // for the next estimate (graph replays)
}

// lambda_it for every it from the moments, the reference's stopping rule, tau
__device__ void circ_final_body(uint32_t NG, const double* Sg, const int* Xg, const double* norm_part,
                                int norm_blocks, double step_safety, double* out) {
    __shared__ double S[kCircMoments];
    __shared__ int X[kCircMoments];
    __shared__ double lam[200];
    __shared__ int first_stop;
    __shared__ double nv2;
    const int t = threadIdx.x;
    if (t == 0) first_stop = 1 << 30;
    for (int p = t; p < kCircMoments; p += 256) {
        S[p] = __ldcg(Sg + p);
        X[p] = __ldcg(Xg + p);
    }
    __shared__ double red[256];
    double s = 0.0;
    for (int b = t; b < norm_blocks; b += 256) s += norm_part[b];
    red[t] = s;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (t < k) red[t] += red[t + k];
        __syncthreads();
    }
    if (t == 0) nv2 = red[0];
    __syncthreads();
    // lambda_0 = mu_1 / |v0|^2 (v0 normalised over all n), lambda_it = mu_2it+1 / mu_2it
    // (solver.cpp:84-86); mu_p = S_p 2^X_p / NG
    if (t < 200) {
        double l;
        if (t == 0)
            l = scalbn(S[1], X[1]) / (static_cast<double>(NG) * nv2);
        else
            l = S[2 * t] != 0.0 ? scalbn(S[2 * t + 1] / S[2 * t], X[2 * t + 1] - X[2 * t]) : 0.0;
        lam[t] = l;
    }
    __syncthreads();
    if (t < 200) {  // the first it at which the reference stops (solver.cpp:88-95)
        const bool zero = S[2 * t + 2] == 0.0;  // M v_it = 0: the zero-operator sentinel
        const bool conv = t > 0 && fabs(lam[t] - lam[t - 1]) <= 1e-6 * fabs(lam[t]);
        if (zero || conv) atomicMin(&first_stop, t);
    }
    __syncthreads();
    if (t == 0) {
        const int it = first_stop < 200 ? first_stop : 199;
        const bool zero = first_stop < 200 && S[2 * it + 2] == 0.0;
        const double l = lam[it];
        out[0] = (zero || l <= 0.0) ? 1.0 : 1.0 / (l * step_safety);  // OUT_TAU
        out[1] = it + 1;                                              // OUT_TAU_ITERS
        out[5] = l;                                                   // OUT_LAMBDA_MAX
        out[6] = 0;  // OUT_TAU_STEPS: no full-operator products
    }
}

// ----------------------------------------------------------------------------- spectral FISTA
// The iterations of run_pgd (solver.cpp:119-151) for a translation-invariant operator, with the
// gradient Theta^T (Theta y - x0) = G y - b applied in the Fourier domain of the translation
// group: (G y)^_f = G_f y^_f, G_f = Theta^_f^H Theta^_f (nCo x nCo, circ_gram_kernel), b = Theta^T x0
// computed once from the representative rows. All arithmetic fp64 (the prox / momentum /
// threshold expressions of the reference, solver.cpp:57-67,126,145).
//
// Grid: g spectral CTAs (g = g0 = g1) + the remaining SMs' CTAs for the decoupled coordinates
// (empty Theta column: prox + momentum only, fp64, run concurrently). Spectral CTA c owns row
// h0 = c of every column orbit (nCo x g coordinates: y, x_prev, p, thr, b in shared memory) and
// column f1 = c of the spectrum (the g blocks G_(f0, c) in shared memory). Per iteration:
//   row phase    (CTA r) inverse row DFTs of T2[.][r][.] -> G y on row r; prox + momentum;
//                forward row DFTs of the new y -> T1[.][r][.]                      -- barrier --
//   column phase (CTA c) column DFTs of T1[.][.][c] -> y^_(f0, c); a^ = G_f y^; inverse column
//                DFTs -> T2[.][.][c]                                                 -- barrier --
// Radix-2 FFTs in shared memory, twiddles e^{2 pi i k / g} from the host (long double).
struct CircFistaArgs {
    const double* x0_full;
    const double* w_full;
    const double* p_full;
    double* x_full;
    const uint32_t* isC;
    uint64_t n;
    const double* beta64;
    double lambda;
    int K;
    const double* out;  // tau at out[0]
    const double2* gram;
    const int* hidx;  // frequency -> half-spectrum index (>= 0) or -1 - index of its conjugate
    const CircOrbit* corb;
    const CircOrbit* rorb;
    const uint32_t* eoff;
    const uint32_t* eh;
    const double* eval;
    const double2* tw;  // e^{+2 pi i k / g}, k < g
    double2* T1;        // [nCo][f1][h0]: row DFTs of y
    double2* T2;        // [nCo][h0][f1]: inverse column DFTs of G_f y^
    unsigned* counter;
    uint32_t g, lg, nRo, nCo, NB;
    uint32_t nimg;  // images in this launch (C5 batches): NB spectral CTAs, T1/T2 and a counter per image
    int staged;     // untracked single-kernel solves: exchange blocks staged in shared memory (see below)
    int diag_skip_decoupled;  // WBX_CIRC_DIAG=nodec: time the spectral CTAs alone (wrong x)
    unsigned long long* prof;  // diagnostics build (WBX_CIRC_PROF=1): CTA 0's cycles per section
    double* outw;              // out (iteration count)
    // energy / support tracking (TRACK instances): per-CTA partials of the spectral CTAs,
    // [k][NB]: q = x_k . G x_k - 2 x_k . b (k = 0..K), r = lambda sum w |x_k|, s = support (k = 1..K);
    // per-warp partials of the decoupled CTAs, [k - 1][nwd]: sum w |x_k| and support; [2][nwd]:
    // sum x0^2 and sum w |x0| over all n
    double* q_part;
    double* r_part;
    double* s_part;
    double* dec_reg;
    double* dec_sup;
    double* e0_part;
    uint32_t nwd;
};


__device__ __forceinline__ void circ_barrier(unsigned* cnt, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.gpu;\nred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        unsigned v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
            if (static_cast<int>(v - target) >= 0) break;
            __nanosleep(32);  // fewer polls contending with the arrivals at the counter's L2 slice
        }
    }
    __syncthreads();
}

// solver.cpp:61-64 (thr = tau * lambda * w / p left to right) and :145
__device__ __forceinline__ double circ_thr(double tau, double lambda, double w, double p) {
    return __ddiv_rn(__dmul_rn(__dmul_rn(tau, lambda), w), p);
}
__device__ __forceinline__ double circ_prox(double z0, double thr) {
    const double a = __dsub_rn(fabs(z0), thr);
    return a > 0.0 ? copysign(a, z0) : 0.0;  // (a > 0 needs |z0| > thr >= 0: z0 != 0, so the sign is z0's)
}
// x' == 0 && x_prev == 0 (either zero sign) by the bits: no fp64 compares in the decoupled loops
__device__ __forceinline__ bool circ_both_zero(double a, double b) {
    return ((static_cast<unsigned long long>(__double_as_longlong(a)) |
             static_cast<unsigned long long>(__double_as_longlong(b))) << 1) == 0;
}
__device__ __forceinline__ double circ_momentum(double xn, double xp, double beta) {
    return __dadd_rn(xn, __dmul_rn(beta, __dsub_rn(xn, xp)));
}


// Warp FFTs of one length-G row held in registers: lane l holds elements l + 32 q (q < PPL).
// DIF forward (e^{-}): natural-order input, bit-reversed-order output; DIT inverse (e^{+}):
// bit-reversed input, natural output (unnormalised). Butterflies of distance d < 32 exchange
// with lane l ^ d by shuffles; d = 32 (G = 64) is lane-local. tw is the per-stage table
// (circ_stage_twiddles): tw[d - 1 + k] = e^{+2 pi i k / (2 d)}, k < d, so the lanes of a stage
// read consecutive entries (no bank conflicts) and tw[d - 1] = 1.
// the per-stage twiddle table of WarpFft from e^{+2 pi i k / G} (k < G): G - 1 entries
template <int G>
__device__ __forceinline__ void circ_stage_twiddles(const double2* __restrict__ twg, double2* tw) {
    for (int i = threadIdx.x; i < G - 1; i += blockDim.x) {
        const int d = 1 << (31 - __clz(i + 1));  // stage of entry i: d - 1 <= i < 2 d - 1
        tw[i] = twg[(i - (d - 1)) * (G / (2 * d))];
    }
}

template <int G>
struct WarpFft {
    static constexpr int PPL = G > 32 ? G / 32 : 1;
    __device__ static double2 shfl(double2 v, int d) {
        return make_double2(__shfl_xor_sync(0xffffffffu, v.x, d), __shfl_xor_sync(0xffffffffu, v.y, d));
    }
    __device__ static void forward(double2 (&v)[PPL], const double2* tw) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int d = G / 2; d >= 1; d >>= 1) {
            if (d >= 32) {  // lane-local: elements lane, lane + 32
                const double2 a = v[0], b = v[1];
                double2 w = tw[d - 1 + lane % d];
                w.y = -w.y;
                v[0] = make_double2(a.x + b.x, a.y + b.y);
                v[1] = cmul(make_double2(a.x - b.x, a.y - b.y), w);
            } else {  // branch free: lo lanes a + b (times tw[0] = 1), hi lanes (a - b) w
                const bool hi = (lane & d) != 0;
#pragma unroll
                for (int q = 0; q < PPL; ++q) {
                    const int e = lane + 32 * q;
                    const double2 p = shfl(v[q], d);
                    double2 w = tw[d - 1 + (hi ? e % d : 0)];
                    w.y = -w.y;
                    const double sg = hi ? -1.0 : 1.0;
                    const double2 r = make_double2(fma(sg, v[q].x, p.x), fma(sg, v[q].y, p.y));
                    v[q] = d == 1 ? r : cmul(r, w);  // the last stage's twiddles are all 1
                }
            }
        }
    }
    __device__ static void inverse(double2 (&v)[PPL], const double2* tw) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int d = 1; d <= G / 2; d <<= 1) {
            if (d >= 32) {
                const double2 w = tw[d - 1 + lane % d];
                const double2 a = v[0], bw = cmul(v[1], w);
                v[0] = make_double2(a.x + bw.x, a.y + bw.y);
                v[1] = make_double2(a.x - bw.x, a.y - bw.y);
            } else {  // branch free: hi lanes pass b w, lo lanes a (times tw[0] = 1)
                const bool hi = (lane & d) != 0;
#pragma unroll
                for (int q = 0; q < PPL; ++q) {
                    const int e = lane + 32 * q;
                    const double2 t = d == 1 ? v[q] : cmul(v[q], tw[d - 1 + (hi ? e % d : 0)]);  // (stage 1: all 1)
                    const double2 p = shfl(t, d);
                    const double sg = hi ? -1.0 : 1.0;
                    v[q] = make_double2(fma(sg, t.x, p.x), fma(sg, t.y, p.y));
                }
            }
        }
    }
};

// The decoupled coordinates of a batch (empty Theta column: gradient exactly 0, so x' = prox(y),
// y = x' + beta (x' - x_prev), solver.cpp:126-145, iterated in registers to the fixed point
// x' == x_prev == 0 or the iteration count) for nimg images back to back, as its own
// full-occupancy launch before the batch's spectral launches: the per-lane trip counts vary
// (0-100 steps), so many resident warps per SM beat the few SMs a batch launch leaves beside
// its spectral CTAs. Same expressions as the in-kernel pass: bitwise the single-image result.
__global__ void __launch_bounds__(256) circ_decoupled_kernel(const double* __restrict__ x0_full,
                                                             double* __restrict__ x_full,
                                                             const double* __restrict__ w_full,
                                                             const double* __restrict__ p_full,
                                                             const uint32_t* __restrict__ isC, uint64_t n, uint32_t nimg,
                                                             const double* __restrict__ beta64, double lambda, int K,
                                                             const double* __restrict__ out) {
    const double tau = out[0];
    const uint64_t total = n * nimg, nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += nthreads) {
        const uint64_t im = t / n, i = t - im * n;
        if ((isC[i >> 5] >> (i & 31)) & 1u) continue;
        const double thr = circ_thr(tau, lambda, w_full[i], p_full[i]);
        double x = x0_full[t], xp = x, y = x;
        for (int k = 1; k <= K; ++k) {
            const double xn = circ_prox(y, thr);
            const bool fixed = circ_both_zero(xn, xp);
            y = circ_momentum(xn, xp, beta64[k - 1]);
            xp = xn;
            x = xn;
            if (fixed) break;
        }
        x_full[t] = x;
    }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}


template <int G>
__device__ __forceinline__ int brev_g(int i) {
    return static_cast<int>(__brev(static_cast<unsigned>(i)) >> (32 - __builtin_ctz(G)));
}

// One CTA per SM: blockIdx < g the spectral CTAs (NCP warps, warp j = orbit row j), the rest the
// decoupled coordinates.
template <int G, int NCP, bool TRACK>
__global__ void __launch_bounds__(32 * NCP, 1) circ_fista_kernel(CircFistaArgs a) {
    using F = WarpFft<G>;
    constexpr int PPL = F::PPL;
    const double tau = a.out[0];
    if (TRACK && blockIdx.x >= a.NB) {
        // decoupled coordinates with their per-iteration sums of w |x_k| and support (warp sums,
        // accumulated over this warp's coordinate trips in a fixed order), and the constant parts
        // of the energies (sum x0^2, sum w |x0| over every coordinate)
        const uint64_t nthreads = static_cast<uint64_t>(gridDim.x - a.NB) * blockDim.x;
        const uint64_t gthread = static_cast<uint64_t>(blockIdx.x - a.NB) * blockDim.x + threadIdx.x;
        const uint32_t gwarp = static_cast<uint32_t>(gthread >> 5);
        const int lane = threadIdx.x & 31;
        double x0sq = 0.0, wx0 = 0.0;
        const uint64_t trips = (a.n + nthreads - 1) / nthreads;  // warp-uniform
        for (uint64_t t = 0; t < trips; ++t) {
            const uint64_t i = t * nthreads + gthread;
            const bool in = i < a.n;
            const bool active = in && !((a.isC[i >> 5] >> (i & 31)) & 1u);
            double x = 0.0, xp = 0.0, y = 0.0, thr = 0.0, w = 0.0;
            if (in) {
                const double x0 = a.x0_full[i];
                w = a.w_full[i];
                x0sq += x0 * x0;
                wx0 += w * fabs(x0);
                if (active) {
                    thr = circ_thr(tau, a.lambda, w, a.p_full[i]);
                    x = xp = y = x0;
                }
            }
            bool live = active;
            for (int k = 1; k <= a.K; ++k) {
                double reg = 0.0, sup = 0.0;
                if (live) {
                    const double xn = circ_prox(y, thr);
                    const bool fixed = circ_both_zero(xn, xp);
                    y = circ_momentum(xn, xp, a.beta64[k - 1]);
                    xp = xn;
                    x = xn;
                    reg = w * fabs(xn);
                    sup = xn != 0.0 ? 1.0 : 0.0;
                    if (fixed) live = false;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    reg += __shfl_xor_sync(0xffffffffu, reg, o);
                    sup += __shfl_xor_sync(0xffffffffu, sup, o);
                }
                if (lane == 0) {
                    a.dec_reg[static_cast<uint64_t>(k - 1) * a.nwd + gwarp] += reg;
                    a.dec_sup[static_cast<uint64_t>(k - 1) * a.nwd + gwarp] += sup;
                }
                if (!__any_sync(0xffffffffu, live)) break;
            }
            if (active) a.x_full[i] = x;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            x0sq += __shfl_xor_sync(0xffffffffu, x0sq, o);
            wx0 += __shfl_xor_sync(0xffffffffu, wx0, o);
        }
        if (lane == 0) {
            a.e0_part[gwarp] = x0sq;
            a.e0_part[a.nwd + gwarp] = wx0;
        }
        return;
    }
    const uint32_t NBS = a.NB * a.nimg;  // spectral CTAs: NB per image of the launch
    if (blockIdx.x >= NBS) {  // (single-image launches; batch launches run circ_decoupled_kernel first)
        if (a.diag_skip_decoupled) return;
        // decoupled coordinates (gradient exactly 0): x' = prox(y), y = x' + beta (x' - x_prev),
        // iterated in registers to the fixed point x' == x_prev == 0 or the iteration count
        const uint64_t nthreads = static_cast<uint64_t>(gridDim.x - NBS) * blockDim.x;
        for (uint64_t i = static_cast<uint64_t>(blockIdx.x - NBS) * blockDim.x + threadIdx.x; i < a.n; i += nthreads) {
            if ((a.isC[i >> 5] >> (i & 31)) & 1u) continue;
            const double thr = circ_thr(tau, a.lambda, a.w_full[i], a.p_full[i]);
            double x = a.x0_full[i], xp = x, y = x;
            for (int k = 1; k <= a.K; ++k) {
                const double xn = circ_prox(y, thr);
                const bool fixed = circ_both_zero(xn, xp);
                y = circ_momentum(xn, xp, a.beta64[k - 1]);
                xp = xn;
                x = xn;
                if (fixed) break;
            }
            a.x_full[i] = x;
        }
        return;
    }
    {  // this CTA's image: its coordinates, exchange buffers and barrier counter
        const uint32_t im = blockIdx.x / a.NB;
        const uint64_t ex = 2ull * a.nCo * a.g * a.g;
        a.x0_full += static_cast<uint64_t>(im) * a.n;
        a.x_full += static_cast<uint64_t>(im) * a.n;
        a.T1 += im * ex;
        a.T2 += im * ex;
        a.counter += 32u * im;
    }
    const int nc = static_cast<int>(a.nCo), c = static_cast<int>(blockIdx.x % a.NB), lane = threadIdx.x & 31,
              wj = threadIdx.x >> 5;
    const bool row_live = wj < nc;  // warp-uniform (lanes >= G of a G = 16 row idle in the shuffles)
    const bool lane_live = lane < G;
    constexpr int GS = NCP + 1;  // padded G block rows
    extern __shared__ double2 circ_smem[];
    double2* Gs = circ_smem;                       // [pos][NCP][NCP + 1]: G_(brev(pos), c), zero padded
    double2* X = Gs + G * NCP * GS;                // [NCP][G]: spectrum of the rows at column c (positions)
    double2* Y = X + NCP * G;                      // [NCP][G + 1]: G_f times it (padded rows: the block
                                                   // products' stores down a column hit distinct banks)
    double2* tw = Y + NCP * (G + 1);               // [G]
    double* ys = reinterpret_cast<double*>(tw + G);  // [NCP][G] y on row c
    double* xps = ys + NCP * G;
    double* bs = xps + NCP * G;
    double* ps = bs + NCP * G;  // tau / p
    double* ths = ps + NCP * G;
    double* gxs = ths + NCP * G;  // TRACK: G x_k-1 on row c (G x_k by linearity from G y_k+1)
    __shared__ double tr_red[3][NCP];  // TRACK: block partials (fixed order)
    // TRACK: this CTA's partials of x . G x - 2 x . b (energy of x_k-1, kq = k - 1) and of
    // lambda w |x| and the support (of x_k, kr = k), summed over its coordinates in a fixed order
    auto track_partials = [&](double q, double r, double sp, int kq, int kr) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            q += __shfl_xor_sync(0xffffffffu, q, o);
            r += __shfl_xor_sync(0xffffffffu, r, o);
            sp += __shfl_xor_sync(0xffffffffu, sp, o);
        }
        if (lane == 0) {
            tr_red[0][wj] = q;
            tr_red[1][wj] = r;
            tr_red[2][wj] = sp;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t[3] = {0.0, 0.0, 0.0};
            for (int w = 0; w < NCP; ++w)
                for (int v = 0; v < 3; ++v) t[v] += tr_red[v][w];
            if (kq >= 0) a.q_part[static_cast<uint64_t>(kq) * a.NB + c] = t[0];
            if (kr >= 1) {
                a.r_part[static_cast<uint64_t>(kr - 1) * a.NB + c] = t[1];
                a.s_part[static_cast<uint64_t>(kr - 1) * a.NB + c] = t[2];
            }
        }
    };
    circ_stage_twiddles<G>(a.tw, tw);
    for (int i = threadIdx.x; i < NCP * (2 * G + 1); i += blockDim.x) X[i] = make_double2(0.0, 0.0);  // padded rows stay 0
    batched_copy(
        G * NCP * NCP,
        [&](uint32_t i) {  // G_(f0, c) for f0 = brev(pos); conjugate half from its partner's block
            const int pos = i / (NCP * NCP), e = i % (NCP * NCP), ii = e / NCP, j = e % NCP;
            if (ii >= nc || j >= nc) return make_double2(0.0, 0.0);
            const int h = a.hidx[brev_g<G>(pos) * G + c];
            const double2 v = a.gram[static_cast<uint64_t>(h >= 0 ? h : -1 - h) * nc * nc + ii * nc + j];
            return h >= 0 ? v : make_double2(v.x, -v.y);
        },
        [&](uint32_t i, double2 v) {
            const int pos = i / (NCP * NCP), e = i % (NCP * NCP);
            Gs[(pos * NCP + e / NCP) * GS + e % NCP] = v;
        });
    // this thread's block-product outputs (t0, t0 + blockDim) and their G rows, in registers
    constexpr int kOut = (G * NCP + 32 * NCP * 2 - 1) / (32 * NCP * 2);  // rounds of two outputs
    static_assert(kOut == 1, "one round of two block-product outputs per thread");
    const int t0 = threadIdx.x, t1 = threadIdx.x + blockDim.x;
    const bool one = t0 < G * NCP, two = t1 < G * NCP;  // G < 32 leaves threads without outputs
    const int pos0 = one ? t0 / NCP : 0, ii0 = one ? t0 % NCP : 0;
    const int pos1 = two ? t1 / NCP : pos0, ii1 = two ? t1 % NCP : ii0;
    __syncthreads();
    double2 g0r[NCP], g1r[NCP];
#pragma unroll
    for (int j = 0; j < NCP; ++j) {
        g0r[j] = Gs[(pos0 * NCP + ii0) * GS + j];
        g1r[j] = Gs[(pos1 * NCP + ii1) * GS + j];
    }
    for (int i = threadIdx.x; i < NCP * G; i += blockDim.x) {  // own row: y = x_prev = x0, p, thr, b
        const int j = i / G, h1 = i % G;
        if (j >= nc) {
            ys[i] = xps[i] = bs[i] = ths[i] = 0.0;
            ps[i] = 1.0;
            continue;
        }
        const CircOrbit o = a.corb[j];
        const uint64_t fl = static_cast<uint64_t>(o.off) + static_cast<uint64_t>(o.a0 + o.s0 * c) * o.W + o.a1 + o.s1 * h1;
        const double x0 = a.x0_full[fl], p = a.p_full[fl];
        ys[i] = x0;
        xps[i] = x0;
        ps[i] = tau / p;
        ths[i] = circ_thr(tau, a.lambda, a.w_full[fl], p);
        // b_j[c][h1] = sum over rows o' and entries (j, e) of its representative: val x0_o'[(c, h1) - e]
        double b = 0.0;
        for (uint32_t r = 0; r < a.nRo; ++r) {
            const CircOrbit ro = a.rorb[r];
            for (uint32_t e = a.eoff[r * nc + j]; e < a.eoff[r * nc + j + 1]; ++e) {
                const uint32_t h = a.eh[e];
                const uint32_t t0 = (c + G - (h >> 16)) & (G - 1), t1 = (h1 + G - (h & 0xffffu)) & (G - 1);
                const uint64_t rf = static_cast<uint64_t>(ro.off) + static_cast<uint64_t>(ro.a0 + ro.s0 * t0) * ro.W +
                                    ro.a1 + ro.s1 * t1;
                b = fma(a.eval[e], a.x0_full[rf], b);
            }
        }
        bs[i] = b;
    }
    __syncthreads();
    const double inv_ng = 1.0 / (static_cast<double>(G) * G);  // exact (power of two)
    unsigned bar = 0;
    // Staged exchange (untracked): T1 as [f1][r][j] and T2 as [h0][c][i] blocks, so a CTA's
    // outputs for one consumer are nc contiguous values (stored from a shared-memory stage by
    // consecutive threads: a few line requests per warp instead of 32 scattered 16-byte
    // sectors) and a consumer's input is one contiguous nc x G block (landed with cp.async).
    // The stage / landing buffer L [G][NCP + 1] reuses the G_f staging (dead after the prologue);
    // its rows are padded so the column reads of a warp (one orbit) are conflict free.
    const bool staged = !TRACK && a.staged;
    constexpr int LP = NCP + 1;
    double2* const L = Gs;
    const uint64_t ncs = a.nCo;
    auto store_T1 = [&]() {  // all threads: L[p][i] (spectrum at f1 = brev(p), orbit i) -> T1[f1][c][i]
        __syncthreads();
        for (int t = threadIdx.x; t < G * nc; t += blockDim.x) {
            const int p = t / nc, i = t - p * nc;
            a.T1[(static_cast<uint64_t>(brev_g<G>(p)) * G + c) * ncs + i] = L[p * LP + i];
        }
    };
    // forward row DFT of this warp's row of y -> T1[j][f1][c] (f1 = brev(position)); staged: -> L
    auto row_forward = [&]() {
        if (!row_live) return;
        double2 v[PPL];
#pragma unroll
        for (int q = 0; q < PPL; ++q) v[q] = make_double2(lane_live ? ys[wj * G + lane + 32 * q] : 0.0, 0.0);
        F::forward(v, tw);
        if (lane_live)
#pragma unroll
            for (int q = 0; q < PPL; ++q) {
                if (staged)
                    L[(lane + 32 * q) * LP + wj] = v[q];
                else
                    a.T1[(static_cast<uint64_t>(wj) * G + brev_g<G>(lane + 32 * q)) * G + c] = v[q];
            }
    };
#if WBX_CIRC_PROF
    __shared__ unsigned long long prof_acc[8];
    if (threadIdx.x < 8) prof_acc[threadIdx.x] = 0;
    __syncthreads();
    long long t_prev = clock64();
    auto mark = [&](int slot) {
        __syncthreads();
        const long long t = clock64();
        if (threadIdx.x == 0) prof_acc[slot] += static_cast<unsigned long long>(t - t_prev);
        t_prev = t;
    };
#else
    auto mark = [](int) {};
#endif
    if (a.K > 0) {
        row_forward();
        if (staged) store_T1();
    }
    for (int k = 1; k <= a.K; ++k) {
        mark(0);
        circ_barrier(a.counter, ++bar * a.NB);
        mark(1);
        if (staged) {  // land T1[f1 = c][r][j] -> L[r][j]
            for (int t = threadIdx.x; t < G * nc; t += blockDim.x) {
                const int r = t / nc, j = t - r * nc;
                cp_async16(L + r * LP + j, a.T1 + (static_cast<uint64_t>(c) * G + r) * ncs + j);
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
            __syncthreads();
        }
        // column phase: column c of the spectrum; warp j transforms orbit j along h0
        if (row_live) {
            double2 v[PPL];
#pragma unroll
            for (int q = 0; q < PPL; ++q)
                v[q] = !lane_live ? make_double2(0.0, 0.0)
                       : staged   ? L[(lane + 32 * q) * LP + wj]
                                  : a.T1[(static_cast<uint64_t>(wj) * G + c) * G + lane + 32 * q];
            F::forward(v, tw);
            if (lane_live)
#pragma unroll
                for (int q = 0; q < PPL; ++q) X[wj * G + lane + 32 * q] = v[q];
        }
        mark(2);
        __syncthreads();
        {  // Y[i][pos] = G_(f0(pos), c) X[.][pos]: two outputs per thread, G rows in registers
            double r0 = 0.0, i0 = 0.0, r1 = 0.0, i1 = 0.0;
#pragma unroll
            for (int j = 0; j < NCP; ++j) {
                const double2 m = g0r[j], x = X[j * G + pos0], n = g1r[j], y = X[j * G + pos1];
                r0 = fma(m.x, x.x, fma(-m.y, x.y, r0));
                i0 = fma(m.x, x.y, fma(m.y, x.x, i0));
                r1 = fma(n.x, y.x, fma(-n.y, y.y, r1));
                i1 = fma(n.x, y.y, fma(n.y, y.x, i1));
            }
            if (one) Y[ii0 * (G + 1) + pos0] = make_double2(r0, i0);
            if (two) Y[ii1 * (G + 1) + pos1] = make_double2(r1, i1);
        }
        mark(3);
        __syncthreads();
        if (row_live) {  // inverse along h0 (bit-reversed positions in, natural h0 out) -> T2[i][h0][c]
            double2 v[PPL];
#pragma unroll
            for (int q = 0; q < PPL; ++q) v[q] = lane_live ? Y[wj * (G + 1) + lane + 32 * q] : make_double2(0.0, 0.0);
            F::inverse(v, tw);
            if (lane_live)
#pragma unroll
                for (int q = 0; q < PPL; ++q) {
                    if (staged)
                        L[(lane + 32 * q) * LP + wj] = v[q];
                    else
                        a.T2[(static_cast<uint64_t>(wj) * G + lane + 32 * q) * G + c] = v[q];
                }
        }
        if (staged) {  // L[h0][i] -> T2[h0][c][i]
            __syncthreads();
            for (int t = threadIdx.x; t < G * nc; t += blockDim.x) {
                const int h0 = t / nc, i = t - h0 * nc;
                a.T2[(static_cast<uint64_t>(h0) * G + c) * ncs + i] = L[h0 * LP + i];
            }
        }
        mark(4);
        circ_barrier(a.counter, ++bar * a.NB);
        mark(5);
        if (staged) {  // land T2[h0 = c][c'][i] -> L[brev(c')][i] (the bit-reversed order the inverse wants)
            for (int t = threadIdx.x; t < G * nc; t += blockDim.x) {
                const int cc = t / nc, i = t - cc * nc;
                cp_async16(L + brev_g<G>(cc) * LP + i, a.T2 + (static_cast<uint64_t>(c) * G + cc) * ncs + i);
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
            __syncthreads();
        }
        // row phase: row c; warp i inverts orbit i along f1 (loaded in bit-reversed order)
        double tq = 0.0, trg = 0.0, tsp = 0.0;  // TRACK partials of this thread
        if (row_live) {
            double2 v[PPL];
#pragma unroll
            for (int q = 0; q < PPL; ++q)
                v[q] = !lane_live ? make_double2(0.0, 0.0)
                       : staged   ? L[(lane + 32 * q) * LP + wj]
                                  : a.T2[(static_cast<uint64_t>(wj) * G + c) * G + brev_g<G>(lane + 32 * q)];
            F::inverse(v, tw);  // v[q].x * NG = (Theta^T Theta y)[wj][c][lane + 32 q]
            const double beta = a.beta64[k - 1];
            const double bprev = k >= 2 ? a.beta64[k - 2] : 0.0;  // y_k = x_k-1 + bprev (x_k-1 - x_k-2)
#pragma unroll
            for (int q = 0; q < PPL; ++q) {
                if (!lane_live) break;
                const int i = wj * G + lane + 32 * q;
                const double gy = v[q].x * inv_ng;                                       // (G y_k)_i
                if constexpr (TRACK) {  // G x_k-1 = (G y_k + bprev G x_k-2) / (1 + bprev); x_k-1 = x_prev
                    const double gx = k == 1 ? gy : (gy + bprev * gxs[i]) / (1.0 + bprev);
                    gxs[i] = gx;
                    tq += xps[i] * (gx - 2.0 * bs[i]);
                }
                const double grad = __dsub_rn(gy, bs[i]);                                 // Theta^T (Theta y - x0)
                const double z0 = fma(-ps[i], grad, ys[i]);  // y - tau g / p (solver.cpp:126), tau / p once
                const double xn = circ_prox(z0, ths[i]);
                ys[i] = circ_momentum(xn, xps[i], beta);
                xps[i] = xn;
                if constexpr (TRACK) {
                    trg += ths[i] / ps[i] * fabs(xn);  // lambda w |x_k|  (thr / (tau / p) = lambda w)
                    tsp += xn != 0.0 ? 1.0 : 0.0;
                }
            }
            __syncwarp();
            if (TRACK || k < a.K) row_forward();
        }
        if (staged && k < a.K) store_T1();
        if constexpr (TRACK) track_partials(tq, trg, tsp, k - 1, k);
        mark(6);
    }
    if (TRACK && a.K > 0) {  // one more column / row pass: G y_K+1 -> G x_K -> the energy of x_K
        circ_barrier(a.counter, ++bar * a.NB);
        if (row_live) {
            double2 v[PPL];
#pragma unroll
            for (int q = 0; q < PPL; ++q)
                v[q] = lane_live ? a.T1[(static_cast<uint64_t>(wj) * G + c) * G + lane + 32 * q] : make_double2(0.0, 0.0);
            F::forward(v, tw);
            if (lane_live)
#pragma unroll
                for (int q = 0; q < PPL; ++q) X[wj * G + lane + 32 * q] = v[q];
        }
        __syncthreads();
        {
            double r0 = 0.0, i0 = 0.0, r1 = 0.0, i1 = 0.0;
#pragma unroll
            for (int j = 0; j < NCP; ++j) {
                const double2 m = g0r[j], x = X[j * G + pos0], n = g1r[j], y = X[j * G + pos1];
                r0 = fma(m.x, x.x, fma(-m.y, x.y, r0));
                i0 = fma(m.x, x.y, fma(m.y, x.x, i0));
                r1 = fma(n.x, y.x, fma(-n.y, y.y, r1));
                i1 = fma(n.x, y.y, fma(n.y, y.x, i1));
            }
            if (one) Y[ii0 * (G + 1) + pos0] = make_double2(r0, i0);
            if (two) Y[ii1 * (G + 1) + pos1] = make_double2(r1, i1);
        }
        __syncthreads();
        if (row_live) {
            double2 v[PPL];
#pragma unroll
            for (int q = 0; q < PPL; ++q) v[q] = lane_live ? Y[wj * (G + 1) + lane + 32 * q] : make_double2(0.0, 0.0);
            F::inverse(v, tw);
            if (lane_live)
#pragma unroll
                for (int q = 0; q < PPL; ++q) a.T2[(static_cast<uint64_t>(wj) * G + lane + 32 * q) * G + c] = v[q];
        }
        circ_barrier(a.counter, ++bar * a.NB);
        double tq = 0.0;
        if (row_live) {
            double2 v[PPL];
#pragma unroll
            for (int q = 0; q < PPL; ++q)
                v[q] = lane_live ? a.T2[(static_cast<uint64_t>(wj) * G + c) * G + brev_g<G>(lane + 32 * q)]
                                 : make_double2(0.0, 0.0);
            F::inverse(v, tw);
            const double bk = a.beta64[a.K - 1];
#pragma unroll
            for (int q = 0; q < PPL; ++q) {
                if (!lane_live) break;
                const int i = wj * G + lane + 32 * q;
                const double gx = (v[q].x * inv_ng + bk * gxs[i]) / (1.0 + bk);
                tq += xps[i] * (gx - 2.0 * bs[i]);
            }
        }
        track_partials(tq, 0.0, 0.0, a.K, 0);
    }
    __syncthreads();
    if (c == 0 && threadIdx.x == 0) a.outw[2] = a.K;  // OUT_ITERS_USED (tracking may lower it)
#if WBX_CIRC_PROF
    if (c == 0 && threadIdx.x < 8) a.prof[threadIdx.x] = prof_acc[threadIdx.x];
#endif
    for (int i = threadIdx.x; i < nc * G; i += blockDim.x) {  // x_final on row c
        const int j = i / G, h1 = i % G;
        const CircOrbit o = a.corb[j];
        a.x_full[static_cast<uint64_t>(o.off) + static_cast<uint64_t>(o.a0 + o.s0 * c) * o.W + o.a1 + o.s1 * h1] = xps[i];
    }
}

template <int G, int NCP>
size_t circ_fista_smem() {
    return static_cast<size_t>(G) * NCP * (NCP + 1) * 16 + NCP * (2 * G + 1) * 16 + G * 16 + 6 * NCP * G * 8;
}

// M images per spectral CTA (C5 batches, untracked): the G_f block rows live in registers
// after the prologue, so the shared memory that staged them holds the state of M images (X, Y,
// y, x_prev, b each) and one grid barrier per phase serves all M. CTA (slot s, column c) owns
// images s M .. s M + M - 1 of the launch; each warp's rows of all M images are fetched with
// cp.async before the first transform, so a phase pays one L2 round trip, not M. Per image the
// arithmetic is circ_fista_kernel's in the same order: bitwise its single-image result. The
// decoupled coordinates run in circ_decoupled_kernel before the launch.
template <int G, int NCP>
__host__ __device__ constexpr int circ_multi_xb() {  // complex values of X and of Y per image
    return NCP * (G + 1) > G * (NCP + 1) ? NCP * (G + 1) : G * (NCP + 1);
}
template <int G, int NCP, int M>
__host__ __device__ constexpr size_t circ_multi_image_bytes() {  // X, Y (complex) + y, x_prev, b
    return static_cast<size_t>(circ_multi_xb<G, NCP>()) * 2 * 16 + static_cast<size_t>(NCP) * G * 3 * 8;
}
template <int G, int NCP, int M>
__host__ __device__ constexpr size_t circ_multi_state_bytes() {
    return static_cast<size_t>(G) * NCP * (NCP + 1) * 16 > M * circ_multi_image_bytes<G, NCP, M>()
               ? static_cast<size_t>(G) * NCP * (NCP + 1) * 16
               : M * circ_multi_image_bytes<G, NCP, M>();
}
template <int G, int NCP, int M>
size_t circ_multi_smem() {  // state (aliasing the G_f staging) + twiddles + tau / p + thresholds
    return circ_multi_state_bytes<G, NCP, M>() + G * 16 + 2 * NCP * G * 8;
}


template <int G, int NCP, int M>
__global__ void __launch_bounds__(32 * NCP, 1) circ_fista_multi_kernel(CircFistaArgs a) {
    using F = WarpFft<G>;
    constexpr int PPL = F::PPL;
    const double tau = a.out[0];
    const uint32_t slots = a.nimg / M;
    if (blockIdx.x >= a.NB * slots) return;
    const uint32_t slot = blockIdx.x / a.NB;
    const int nc = static_cast<int>(a.nCo), c = static_cast<int>(blockIdx.x % a.NB), lane = threadIdx.x & 31,
              wj = threadIdx.x >> 5;
    const bool row_live = wj < nc;
    const bool lane_live = lane < G;
    const uint64_t ex = 2ull * a.nCo * a.g * a.g;  // T1, T2 per image
    unsigned* const counter = a.counter + 32u * slot;
    constexpr int GS = NCP + 1;
    constexpr size_t kImg = circ_multi_image_bytes<G, NCP, M>();
    extern __shared__ double2 circ_smem[];
    unsigned char* const sbase = reinterpret_cast<unsigned char*>(circ_smem);
    double2* Gs = circ_smem;  // prologue only; then the images' state
    double2* tw = reinterpret_cast<double2*>(sbase + circ_multi_state_bytes<G, NCP, M>());
    double* ps = reinterpret_cast<double*>(tw + G);  // tau / p (the images share P, w, lambda, tau)
    double* ths = ps + NCP * G;
    // X, Y of an image: [NCP][G] spectra / [NCP][G + 1] block products, and (staged exchange, as
    // circ_fista_kernel) [G][NCP + 1] landing / stage blocks: XB complex values each
    constexpr int LP = NCP + 1;
    constexpr int XB = circ_multi_xb<G, NCP>();
    const uint64_t ncs = a.nCo;
    auto Xm = [&](int m) { return reinterpret_cast<double2*>(sbase + m * kImg); };
    auto Ym = [&](int m) { return Xm(m) + XB; };
    auto ysm = [&](int m) { return reinterpret_cast<double*>(Ym(m) + XB); };
    auto xpm = [&](int m) { return ysm(m) + NCP * G; };
    auto bsm = [&](int m) { return xpm(m) + NCP * G; };
    auto img = [&](int m) { return static_cast<uint64_t>(slot) * M + m; };
    circ_stage_twiddles<G>(a.tw, tw);
    batched_copy(
        G * NCP * NCP,
        [&](uint32_t i) {
            const int pos = i / (NCP * NCP), e = i % (NCP * NCP), ii = e / NCP, j = e % NCP;
            if (ii >= nc || j >= nc) return make_double2(0.0, 0.0);
            const int h = a.hidx[brev_g<G>(pos) * G + c];
            const double2 v = a.gram[static_cast<uint64_t>(h >= 0 ? h : -1 - h) * nc * nc + ii * nc + j];
            return h >= 0 ? v : make_double2(v.x, -v.y);
        },
        [&](uint32_t i, double2 v) {
            const int pos = i / (NCP * NCP), e = i % (NCP * NCP);
            Gs[(pos * NCP + e / NCP) * GS + e % NCP] = v;
        });
    constexpr int kOut = (G * NCP + 32 * NCP * 2 - 1) / (32 * NCP * 2);
    static_assert(kOut == 1, "one round of two block-product outputs per thread");
    const int t0 = threadIdx.x, t1 = threadIdx.x + blockDim.x;
    const bool one = t0 < G * NCP, two = t1 < G * NCP;
    const int pos0 = one ? t0 / NCP : 0, ii0 = one ? t0 % NCP : 0;
    const int pos1 = two ? t1 / NCP : pos0, ii1 = two ? t1 % NCP : ii0;
    __syncthreads();
    double2 g0r[NCP], g1r[NCP];
#pragma unroll
    for (int j = 0; j < NCP; ++j) {
        g0r[j] = Gs[(pos0 * NCP + ii0) * GS + j];
        g1r[j] = Gs[(pos1 * NCP + ii1) * GS + j];
    }
    __syncthreads();  // the staging is dead: the images' state takes its place
    for (int m = 0; m < M; ++m)
        for (int i = threadIdx.x; i < 2 * XB; i += blockDim.x) Xm(m)[i] = make_double2(0.0, 0.0);  // X, Y
    for (int i = threadIdx.x; i < NCP * G; i += blockDim.x) {  // own row: p, thr; per image y = x_prev = x0, b
        const int j = i / G, h1 = i % G;
        if (j >= nc) {
            ths[i] = 0.0;
            ps[i] = 1.0;
            for (int m = 0; m < M; ++m) ysm(m)[i] = xpm(m)[i] = bsm(m)[i] = 0.0;
            continue;
        }
        const CircOrbit o = a.corb[j];
        const uint64_t fl = static_cast<uint64_t>(o.off) + static_cast<uint64_t>(o.a0 + o.s0 * c) * o.W + o.a1 + o.s1 * h1;
        const double p = a.p_full[fl];
        ps[i] = tau / p;
        ths[i] = circ_thr(tau, a.lambda, a.w_full[fl], p);
        for (int m = 0; m < M; ++m) {
            const double* x0 = a.x0_full + img(m) * a.n;
            ysm(m)[i] = x0[fl];
            xpm(m)[i] = x0[fl];
            double b = 0.0;  // b_j[c][h1], as circ_fista_kernel
            for (uint32_t r = 0; r < a.nRo; ++r) {
                const CircOrbit ro = a.rorb[r];
                for (uint32_t e = a.eoff[r * nc + j]; e < a.eoff[r * nc + j + 1]; ++e) {
                    const uint32_t h = a.eh[e];
                    const uint32_t q0 = (c + G - (h >> 16)) & (G - 1), q1 = (h1 + G - (h & 0xffffu)) & (G - 1);
                    const uint64_t rf = static_cast<uint64_t>(ro.off) + static_cast<uint64_t>(ro.a0 + ro.s0 * q0) * ro.W +
                                        ro.a1 + ro.s1 * q1;
                    b = fma(a.eval[e], x0[rf], b);
                }
            }
            bsm(m)[i] = b;
        }
    }
    __syncthreads();
    const double inv_ng = 1.0 / (static_cast<double>(G) * G);
    unsigned bar = 0;
    auto row_forward = [&](int m) {  // row DFT of this warp's row of image m's y -> X_m stage [p][j]
        double2 v[PPL];
#pragma unroll
        for (int q = 0; q < PPL; ++q) v[q] = make_double2(lane_live ? ysm(m)[wj * G + lane + 32 * q] : 0.0, 0.0);
        F::forward(v, tw);
        if (lane_live)
#pragma unroll
            for (int q = 0; q < PPL; ++q) Xm(m)[(lane + 32 * q) * LP + wj] = v[q];
    };
    auto store_T1 = [&]() {  // all threads: X_m[p][i] (f1 = brev(p)) -> T1_m[f1][c][i], every image
        __syncthreads();
        for (int m = 0; m < M; ++m) {
            double2* T1 = a.T1 + img(m) * ex;
            for (int t = threadIdx.x; t < G * nc; t += blockDim.x) {
                const int p = t / nc, i = t - p * nc;
                T1[(static_cast<uint64_t>(brev_g<G>(p)) * G + c) * ncs + i] = Xm(m)[p * LP + i];
            }
        }
    };
    if (a.K > 0) {
        if (row_live)
            for (int m = 0; m < M; ++m) row_forward(m);
        store_T1();
    }
    for (int k = 1; k <= a.K; ++k) {
        circ_barrier(counter, ++bar * a.NB);
        // column phase: each image's block T1[f1 = c][r][j] landed in Y [r][j], transformed into X
        for (int m = 0; m < M; ++m) {
            const double2* T1 = a.T1 + img(m) * ex + static_cast<uint64_t>(c) * G * ncs;
            for (int t = threadIdx.x; t < G * nc; t += blockDim.x) {
                const int r = t / nc, j = t - r * nc;
                cp_async16(Ym(m) + r * LP + j, T1 + static_cast<uint64_t>(r) * ncs + j);
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (row_live) {
            for (int m = 0; m < M; ++m) {
                double2 v[PPL];
#pragma unroll
                for (int q = 0; q < PPL; ++q) v[q] = lane_live ? Ym(m)[(lane + 32 * q) * LP + wj] : make_double2(0.0, 0.0);
                F::forward(v, tw);
                if (lane_live)
#pragma unroll
                    for (int q = 0; q < PPL; ++q) Xm(m)[wj * G + lane + 32 * q] = v[q];
            }
        }
        __syncthreads();
        for (int m = 0; m < M; ++m) {  // Y = G_f X per image, the block rows from registers
            const double2* X = Xm(m);
            double r0 = 0.0, i0 = 0.0, r1 = 0.0, i1 = 0.0;
#pragma unroll
            for (int j = 0; j < NCP; ++j) {
                const double2 mm = g0r[j], x = X[j * G + pos0], n = g1r[j], y = X[j * G + pos1];
                r0 = fma(mm.x, x.x, fma(-mm.y, x.y, r0));
                i0 = fma(mm.x, x.y, fma(mm.y, x.x, i0));
                r1 = fma(n.x, y.x, fma(-n.y, y.y, r1));
                i1 = fma(n.x, y.y, fma(n.y, y.x, i1));
            }
            if (one) Ym(m)[ii0 * (G + 1) + pos0] = make_double2(r0, i0);
            if (two) Ym(m)[ii1 * (G + 1) + pos1] = make_double2(r1, i1);
        }
        __syncthreads();
        if (row_live)
            for (int m = 0; m < M; ++m) {  // inverse along h0 -> T2[i][h0][c]
                double2 v[PPL];
#pragma unroll
                for (int q = 0; q < PPL; ++q) v[q] = lane_live ? Ym(m)[wj * (G + 1) + lane + 32 * q] : make_double2(0.0, 0.0);
                F::inverse(v, tw);  // -> X_m stage [h0][i] (the products are done with X)
                if (lane_live)
#pragma unroll
                    for (int q = 0; q < PPL; ++q) Xm(m)[(lane + 32 * q) * LP + wj] = v[q];
            }
        __syncthreads();
        for (int m = 0; m < M; ++m) {  // X_m[h0][i] -> T2_m[h0][c][i]
            double2* T2 = a.T2 + img(m) * ex;
            for (int t = threadIdx.x; t < G * nc; t += blockDim.x) {
                const int h0 = t / nc, i = t - h0 * nc;
                T2[(static_cast<uint64_t>(h0) * G + c) * ncs + i] = Xm(m)[h0 * LP + i];
            }
        }
        circ_barrier(counter, ++bar * a.NB);
        // row phase: each image's block T2[h0 = c][c'][i] landed in X [brev(c')][i] (bit-reversed rows)
        for (int m = 0; m < M; ++m) {
            const double2* T2 = a.T2 + img(m) * ex + static_cast<uint64_t>(c) * G * ncs;
            for (int t = threadIdx.x; t < G * nc; t += blockDim.x) {
                const int cc = t / nc, i = t - cc * nc;
                cp_async16(Xm(m) + brev_g<G>(cc) * LP + i, T2 + static_cast<uint64_t>(cc) * ncs + i);
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (row_live) {
            const double beta = a.beta64[k - 1];
            for (int m = 0; m < M; ++m) {
                double2 v[PPL];
#pragma unroll
                for (int q = 0; q < PPL; ++q) v[q] = lane_live ? Xm(m)[(lane + 32 * q) * LP + wj] : make_double2(0.0, 0.0);
                F::inverse(v, tw);
                double* ys = ysm(m);
                double* xps = xpm(m);
                const double* bs = bsm(m);
#pragma unroll
                for (int q = 0; q < PPL; ++q) {
                    if (!lane_live) break;
                    const int i = wj * G + lane + 32 * q;
                    const double gy = v[q].x * inv_ng;
                    const double grad = __dsub_rn(gy, bs[i]);
                    const double z0 = fma(-ps[i], grad, ys[i]);
                    const double xn = circ_prox(z0, ths[i]);
                    ys[i] = circ_momentum(xn, xps[i], beta);
                    xps[i] = xn;
                }
                __syncwarp();
                if (k < a.K) row_forward(m);
            }
        }
        if (k < a.K) store_T1();
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) a.outw[2] = a.K;  // OUT_ITERS_USED
    for (int m = 0; m < M; ++m) {
        double* x = a.x_full + img(m) * a.n;
        for (int i = threadIdx.x; i < nc * G; i += blockDim.x) {
            const int j = i / G, h1 = i % G;
            const CircOrbit o = a.corb[j];
            x[static_cast<uint64_t>(o.off) + static_cast<uint64_t>(o.a0 + o.s0 * c) * o.W + o.a1 + o.s1 * h1] = xpm(m)[i];
        }
    }
}

// Energies of the tracked spectral solve (run_pgd's E(x_k), solver.cpp:44-55, 118, 130): block k
// sums the partials in a fixed order; E_k = (q_k + |x0|^2) / 2 + lambda sum w |x_k|, with
// |Theta x - x0|^2 = x . G x - 2 x . Theta^T x0 + |x0|^2. Block 0: the initial energy.
__global__ void __launch_bounds__(256) circ_energy_kernel(const double* __restrict__ q_part,
                                                          const double* __restrict__ r_part,
                                                          const double* __restrict__ s_part,
                                                          const double* __restrict__ dec_reg,
                                                          const double* __restrict__ dec_sup,
                                                          const double* __restrict__ e0_part, uint32_t NB, uint32_t nwd,
                                                          double lambda, double* energies,
                                                          unsigned long long* supports, double* out) {
    __shared__ double red[4][256];
    const int k = blockIdx.x, t = threadIdx.x;
    double v[4] = {0.0, 0.0, 0.0, 0.0};  // q + ... , C-part reg, decoupled reg, support
    for (uint32_t i = t; i < NB; i += 256) {
        v[0] += q_part[static_cast<uint64_t>(k) * NB + i];
        if (k >= 1) {
            v[1] += r_part[static_cast<uint64_t>(k - 1) * NB + i];
            v[3] += s_part[static_cast<uint64_t>(k - 1) * NB + i];
        }
    }
    for (uint32_t i = t; i < nwd; i += 256) {
        v[0] += e0_part[i];  // |x0|^2
        if (k >= 1) {
            v[2] += dec_reg[static_cast<uint64_t>(k - 1) * nwd + i];
            v[3] += dec_sup[static_cast<uint64_t>(k - 1) * nwd + i];
        } else {
            v[2] += e0_part[nwd + i];  // sum w |x0|
        }
    }
    for (int j = 0; j < 4; ++j) red[j][t] = v[j];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (t < s)
            for (int j = 0; j < 4; ++j) red[j][t] += red[j][t + s];
        __syncthreads();
    }
    if (t == 0) {
        const double e = 0.5 * red[0][0] + red[1][0] + lambda * red[2][0];
        if (k == 0) {
            out[3] = e;  // OUT_INITIAL_ENERGY
        } else {
            energies[k - 1] = e;
            supports[k - 1] = static_cast<unsigned long long>(red[3][0]);
        }
    }
}

// NonFiniteEnergy (solver.cpp:131-133): the first iteration with a non-finite energy ends the
// solve there (status 8, the host raises)
__global__ void circ_energy_check_kernel(const double* energies, int K, double* out) {
    if (threadIdx.x != 0) return;
    for (int k = 0; k < K; ++k)
        if (!isfinite(energies[k])) {
            out[4] = 8.0;   // OUT_STATUS
            out[2] = k + 1; // OUT_ITERS_USED
            return;
        }
}

// ----------------------------------------------------------------------------- host

double2 twiddle(uint64_t k, uint64_t g) {
    const long double a = 2.0L * 3.14159265358979323846264338327950288L * static_cast<long double>(k) /
                          static_cast<long double>(g);
    return make_double2(static_cast<double>(cosl(a)), static_cast<double>(sinl(a)));
}

}  // namespace

// Host analysis of an operator against a wavelet layout (no device work). ok == false with
// `why` when the operator is not translation invariant or outside the kernel's limits.
std::shared_ptr<CircPlan> circ_analyze(const wbx_op* op, uint32_t ndim, const uint64_t* dims, uint32_t J,
                                       const std::vector<wbx_band>& bands) {
    auto P = std::make_shared<CircPlan>();
    auto no = [&](const std::string& w) {
        P->why = w;
        return P;
    };
    const uint64_t n = op->n;
    P->n = n;
    if (dims[0] * (ndim == 2 ? dims[1] : 1) != n) return no("layout size differs from the operator");
    if (op->h_rowptr.size() != n + 1) return no("no host CSR");
    const uint64_t g0 = dims[0] >> J, g1 = ndim == 2 ? dims[1] >> J : 1;
    if (g0 == 0 || g1 == 0 || (g0 << J) != dims[0] || (ndim == 2 && (g1 << J) != dims[1]))
        return no("dims not divisible by 2^J");
    if (g0 > 1024 || g1 > 1024) return no("translation group larger than 1024 per dimension");
    P->g0 = static_cast<uint32_t>(g0);
    P->g1 = static_cast<uint32_t>(g1);
    P->NG = static_cast<uint32_t>(g0 * g1);
    const uint64_t NG = g0 * g1;
    // orbit / group element of every flat index
    std::vector<uint32_t> orb(n), grp(n);
    std::vector<CircOrbit> orbits;
    std::vector<uint64_t> rep_flat;
    for (const wbx_band& b : bands) {
        const uint64_t sh0 = b.shape[0], sh1 = ndim == 2 ? b.shape[1] : 1;
        if (sh0 % g0 || sh1 % g1) return no("band shape not a multiple of the group");
        const uint64_t s0 = sh0 / g0, s1 = sh1 / g1;
        const uint32_t base = static_cast<uint32_t>(orbits.size());
        for (uint64_t a0 = 0; a0 < s0; ++a0)
            for (uint64_t a1 = 0; a1 < s1; ++a1) {
                orbits.push_back(CircOrbit{static_cast<uint32_t>(b.offset), static_cast<uint32_t>(sh1),
                                           static_cast<uint32_t>(a0), static_cast<uint32_t>(a1),
                                           static_cast<uint32_t>(s0), static_cast<uint32_t>(s1)});
                rep_flat.push_back(b.offset + a0 * sh1 + a1);
            }
        for (uint64_t p0 = 0; p0 < sh0; ++p0)
            for (uint64_t p1 = 0; p1 < sh1; ++p1) {
                const uint64_t fl = b.offset + p0 * sh1 + p1;
                orb[fl] = base + static_cast<uint32_t>((p0 % s0) * s1 + p1 % s1);
                grp[fl] = static_cast<uint32_t>((p0 / s0) * g1 + p1 / s1);
            }
    }
    const auto& rp = op->h_rowptr;
    const auto& ci = op->h_col;
    const auto& va = op->h_val;
    // column orbits holding nonzeros
    std::vector<int32_t> cidx(orbits.size(), -1);
    for (uint64_t e = 0; e < ci.size(); ++e) cidx[orb[ci[e]]] = 0;
    uint32_t nCo = 0;
    for (size_t o = 0; o < orbits.size(); ++o)
        if (cidx[o] == 0) {
            cidx[o] = static_cast<int32_t>(nCo++);
            P->h_orb.push_back(orbits[o]);
            P->c_rep.push_back(static_cast<uint32_t>(rep_flat[o]));
        }
    if (nCo == 0) return no("empty operator");
    if (nCo > static_cast<uint32_t>(kCircMaxCo)) return no("more than 16 column orbits");
    P->nCo = nCo;
    // representative rows; every row must equal its representative shifted by its group element
    auto shift = [&](uint32_t h, uint32_t t) {  // h - t in the group
        const uint64_t a0 = h / g1, a1 = h % g1, b0 = t / g1, b1 = t % g1;
        return static_cast<uint32_t>(((a0 + g0 - b0) % g0) * g1 + (a1 + g1 - b1) % g1);
    };
    std::vector<double> table(static_cast<size_t>(nCo) * NG);
    std::vector<uint8_t> used(static_cast<size_t>(nCo) * NG);
    uint64_t covered = 0;
    std::vector<uint32_t> eoff{0};
    for (size_t o = 0; o < orbits.size(); ++o) {
        const uint64_t r0 = rep_flat[o];
        const uint64_t len = rp[r0 + 1] - rp[r0];
        if (len == 0) continue;
        std::fill(used.begin(), used.end(), 0);
        // entries of the representative grouped by column orbit (CSR order inside a group)
        std::vector<std::vector<uint64_t>> by(nCo);
        for (uint64_t e = rp[r0]; e < rp[r0 + 1]; ++e) {
            const uint32_t j = static_cast<uint32_t>(cidx[orb[ci[e]]]);
            const size_t key = static_cast<size_t>(j) * NG + grp[ci[e]];
            table[key] = va[e];
            used[key] = 1;
            by[j].push_back(e);
        }
        for (uint32_t j = 0; j < nCo; ++j) {
            for (uint64_t e : by[j]) {
                const uint32_t h = grp[ci[e]];
                P->h_eh.push_back(((h / static_cast<uint32_t>(g1)) << 16) | (h % static_cast<uint32_t>(g1)));
                P->h_eval.push_back(va[e]);
            }
            eoff.push_back(static_cast<uint32_t>(P->h_eval.size()));
        }
        // every row of the orbit
        const CircOrbit& ob = orbits[o];
        P->h_rorb.push_back(ob);
        for (uint64_t h0 = 0; h0 < g0; ++h0)
            for (uint64_t h1 = 0; h1 < g1; ++h1) {
                const uint64_t r = ob.off + (ob.a0 + ob.s0 * h0) * ob.W + ob.a1 + ob.s1 * h1;
                if (rp[r + 1] - rp[r] != len) return no("row lengths vary within an orbit");
                const uint32_t t = static_cast<uint32_t>(h0 * g1 + h1);
                for (uint64_t e = rp[r]; e < rp[r + 1]; ++e) {
                    const size_t key = static_cast<size_t>(cidx[orb[ci[e]]]) * NG + shift(grp[ci[e]], t);
                    if (!used[key] || std::memcmp(&table[key], &va[e], sizeof(double)) != 0)
                        return no("operator is not translation invariant");
                }
                covered += len;
            }
        ++P->nRo;
    }
    if (covered != ci.size()) return no("nonzeros outside the representative orbits' rows");
    if (P->nRo == 0) return no("empty operator");
    // the representative rows and twiddles are staged in shared memory by circ_lanczos_kernel
    if (eoff.size() * 4 + P->h_eval.size() * 12 + (g0 + g1) * 16 + 4 * P->nRo * nCo * 16 > 96u * 1024u)
        return no("representative rows too long for shared memory");
    P->h_eoff = std::move(eoff);
    // overflow safety of 4 unnormalised power steps: |M^_f| <= (sum |val|)^2 max(P^-1) is
    // checked per solver (circ_check_p)
    for (uint64_t f0 = 0; f0 < g0; ++f0)  // one of every conjugate pair {f, -f}, weight 2
        for (uint64_t f1 = 0; f1 < g1; ++f1) {
            const uint64_t f = f0 * g1 + f1, fc = ((g0 - f0) % g0) * g1 + (g1 - f1) % g1;
            if (f <= fc) P->h_fhalf.push_back(static_cast<uint32_t>(f << 1 | (f < fc ? 1u : 0u)));
        }
    P->h_hidx.assign(NG, 0);
    for (size_t i = 0; i < P->h_fhalf.size(); ++i) {
        const uint64_t f = P->h_fhalf[i] >> 1, f0 = f / g1, f1 = f % g1;
        const uint64_t fc = ((g0 - f0) % g0) * g1 + (g1 - f1) % g1;
        P->h_hidx[f] = static_cast<int>(i);
        if (fc != f) P->h_hidx[fc] = -1 - static_cast<int>(i);
    }
    for (uint64_t k = 0; k < g0; ++k) P->h_tw0.push_back(twiddle(k, g0));
    for (uint64_t k = 0; k < g1; ++k) P->h_tw1.push_back(twiddle(k, g1));
    P->ok = true;
    // the spectral FISTA engine: square translation group of 16, 32 or 64, its shared memory
    const uint64_t ncp = (nCo + 3) / 4 * 4;
    const uint64_t fista_smem = g0 * ncp * (ncp + 1) * 16 + 2 * ncp * g0 * 16 + g0 * 16 + 6 * ncp * g0 * 8;
    if (ndim != 2 || g0 != g1 || (g0 != 8 && g0 != 16 && g0 != 32 && g0 != 64))
        P->fista_why = "spectral FISTA needs a square translation group of 8, 16, 32 or 64";
    else if (fista_smem > 227u * 1024u)
        P->fista_why = "spectral FISTA blocks exceed shared memory";
    else
        P->fista_ok = true;
    return P;
}

bool circ_plan_ok(const CircPlan& P, std::string* why, uint32_t* info5) {
    if (why) *why = P.why;
    if (info5) {
        info5[0] = P.ok;
        info5[1] = P.nRo;
        info5[2] = P.nCo;
        info5[3] = P.g0;
        info5[4] = P.g1;
    }
    return P.ok;
}

bool circ_fista_ok(const CircPlan& P, std::string* why) {
    if (why) *why = P.ok ? P.fista_why : P.why;
    return P.ok && P.fista_ok;
}

// Per-solver check of P on the column orbits; fills isp (P^-1/2 of each column orbit).
bool circ_check_p(const CircPlan& P, const double* p, std::vector<double>& isp, std::string* why) {
    isp.assign(P.nCo, 0.0);
    double sumv = 0.0;
    for (double v : P.h_eval) sumv += std::fabs(v);
    double maxisp = 0.0;
    for (uint32_t j = 0; j < P.nCo; ++j) {
        const CircOrbit& o = P.h_orb[j];
        const double pr = p[P.c_rep[j]];
        for (uint64_t h0 = 0; h0 < P.g0; ++h0)
            for (uint64_t h1 = 0; h1 < P.g1; ++h1) {
                const uint64_t fl = o.off + (o.a0 + o.s0 * h0) * o.W + o.a1 + o.s1 * h1;
                if (!(std::fabs(p[fl] - pr) <= 1e-12 * std::fabs(pr))) {
                    if (why) *why = "preconditioner not constant on a column orbit";
                    return false;
                }
            }
        isp[j] = 1.0 / std::sqrt(pr);  // solver.cpp:72
        maxisp = std::max(maxisp, isp[j]);
    }
    const double bound = sumv * maxisp;  // |M^_f| <= bound^2; 4 steps grow z by <= bound^8
    if (!(bound > 0.0) || !(std::fabs(std::log2(bound)) * 8.0 < 900.0)) {
        if (why) *why = "operator scale outside the unnormalised power steps' range";
        return false;
    }
    return true;
}

namespace {
struct FistaKernel {
    const void* fn = nullptr;
    size_t smem = 0;
    int warps = 0;
};
template <int G, int NCP>
FistaKernel fista_kernel_of(bool track) {
    return FistaKernel{track ? reinterpret_cast<const void*>(circ_fista_kernel<G, NCP, true>)
                             : reinterpret_cast<const void*>(circ_fista_kernel<G, NCP, false>),
                       circ_fista_smem<G, NCP>(), NCP};
}
template <int G>
FistaKernel fista_kernel_g(uint32_t nc, bool track) {
    if (nc <= 4) return fista_kernel_of<G, 4>(track);
    if (nc <= 8) return fista_kernel_of<G, 8>(track);
    if (nc <= 12) return fista_kernel_of<G, 12>(track);
    return fista_kernel_of<G, 16>(track);
}
// (g, nCo, tracking) -> instance: g in {8, 16, 32, 64}, nCo padded to 4, 8, 12, 16 rows (warps)
FistaKernel fista_kernel_for(uint32_t g, uint32_t nc, bool track = false) {
    if (g == 8) return fista_kernel_g<8>(nc, track);
    if (g == 16) return fista_kernel_g<16>(nc, track);
    if (g == 32) return fista_kernel_g<32>(nc, track);
    if (g == 64) return fista_kernel_g<64>(nc, track);
    return FistaKernel{};
}
// M images per CTA (batches, g = 32, 64: the groups whose images per launch are few); no
// instance when the state does not fit the opt-in shared memory
constexpr size_t kMaxSmem = 227 * 1024;
template <int G, int NCP, int M>
FistaKernel multi_kernel_of() {
    if (circ_multi_smem<G, NCP, M>() > kMaxSmem) return FistaKernel{};
    return FistaKernel{reinterpret_cast<const void*>(circ_fista_multi_kernel<G, NCP, M>), circ_multi_smem<G, NCP, M>(), NCP};
}
template <int G, int M>
FistaKernel multi_kernel_g(uint32_t nc) {
    if (nc <= 4) return multi_kernel_of<G, 4, M>();
    if (nc <= 8) return multi_kernel_of<G, 8, M>();
    if (nc <= 12) return multi_kernel_of<G, 12, M>();
    return multi_kernel_of<G, 16, M>();
}
FistaKernel multi_kernel_for(uint32_t g, uint32_t nc, uint32_t m) {
    if (g == 32) return m == 2 ? multi_kernel_g<32, 2>(nc) : m == 4 ? multi_kernel_g<32, 4>(nc) : FistaKernel{};
    if (g == 64) return m == 2 ? multi_kernel_g<64, 2>(nc) : m == 4 ? multi_kernel_g<64, 4>(nc) : FistaKernel{};
    return FistaKernel{};
}
// images per CTA for a launch of nimg images: 1 while one image per CTA fits the grid, else the
// smallest M in {2, 4} that divides nimg and fits (0: none; WBX_CIRC_MULTI=0 turns them off)
uint32_t multi_m(const CircPlan& P, int num_sms, uint32_t nimg) {
    const uint32_t smax = static_cast<uint32_t>(num_sms) / P.g0;
    if (nimg <= smax) return 1;
    if (const char* e = std::getenv("WBX_CIRC_MULTI"); e && std::string(e) == "0") return 0;
    for (const uint32_t m : {2u, 4u})
        if (nimg % m == 0 && nimg / m <= smax && multi_kernel_for(P.g0, P.nCo, m).fn) return m;
    return 0;
}
}  // namespace

void circ_upload(CircPlan& P, cudaStream_t st) {
    if (P.uploaded) return;
    P.orb.alloc(P.h_orb.size());
    P.orb.upload(P.h_orb.data(), P.h_orb.size(), st);
    P.eoff.upload(P.h_eoff, st);
    P.eh.upload(P.h_eh.empty() ? std::vector<uint32_t>{0} : P.h_eh, st);
    P.eval.upload(P.h_eval.empty() ? std::vector<double>{0.0} : P.h_eval, st);
    P.tw0.upload(P.h_tw0, st);
    P.tw1.upload(P.h_tw1, st);
    P.fhalf.upload(P.h_fhalf, st);
    P.hidx.upload(P.h_hidx, st);
    P.rorb.alloc(P.h_rorb.size());
    P.rorb.upload(P.h_rorb.data(), P.h_rorb.size(), st);
    WBX_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(circ_gram_kernel),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    if (P.fista_ok) {
        for (const bool track : {false, true}) {
            const FistaKernel k = fista_kernel_for(P.g0, P.nCo, track);
            WBX_CUDA(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(k.smem)));
        }
        for (const uint32_t m : {2u, 4u})
            if (const FistaKernel k = multi_kernel_for(P.g0, P.nCo, m); k.fn)
                WBX_CUDA(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(k.smem)));
    }
    WBX_CUDA(cudaStreamSynchronize(st));
    P.uploaded = true;
}

// Work buffers of one solver's estimate (double-sized units)
uint64_t circ_work_doubles(const CircPlan& P) {
    const uint64_t nh = P.h_fhalf.size();
    return kCircNormBlocks + 4ull * P.nCo * P.NG /* t1, vh */ + (2 * kCircMaxCo + 2) * nh /* T_f */ +
           kCircMoments * nh /* mom_m */ +
           (kCircMoments * nh + 1) / 2 /* mom_e */ + kCircMoments /* S */ + (kCircMoments + 1) / 2 /* X */ +
           16 /* done counter (zeroed at allocation, reset by its last block) */;
}

// Enqueue the estimate; writes out[OUT_TAU], out[OUT_TAU_ITERS], out[OUT_LAMBDA_MAX], out[OUT_TAU_STEPS].
// G_f = Theta^_f^H Theta^_f for the half spectrum (nh x nCo x nCo complex)
uint64_t circ_gram_doubles(const CircPlan& P) { return 2ull * P.h_fhalf.size() * P.nCo * P.nCo; }
void circ_gram_launch(wbx_ctx* ctx, const CircPlan& P, double2* gram, cudaStream_t st) {
    const uint32_t nh = static_cast<uint32_t>(P.h_fhalf.size());
    const uint32_t nent = static_cast<uint32_t>(P.h_eval.size());
    const size_t smem = kGramWarps * P.nRo * P.nCo * sizeof(double2) + (P.g0 + P.g1) * sizeof(double2) +
                        nent * (sizeof(double) + sizeof(uint32_t)) + (P.nRo * P.nCo + 1) * sizeof(uint32_t);
    circ_gram_kernel<<<(nh + kGramWarps - 1) / kGramWarps, kGramWarps * 32, smem, st>>>(
        nh, P.fhalf.p, P.g1, P.g0, P.nRo, P.nCo, P.eoff.p, P.eh.p, P.eval.p, P.tw0.p, P.tw1.p, gram, nent);
    count_launch(ctx);
}

// The spectral FISTA engine's exchange buffers T1, T2 (2 x nCo x NG complex)
uint64_t circ_exchange_doubles(const CircPlan& P) { return 4ull * P.nCo * P.NG; }
uint32_t circ_fista_blocks(const CircPlan& P) { return P.g0; }
uint32_t circ_fista_slots(const CircPlan& P, int num_sms, uint32_t batch) {
    // batch launches run no decoupled CTAs (circ_decoupled_kernel takes those coordinates), so
    // every SM can hold a spectral CTA, and M images per CTA (circ_fista_multi_kernel) when one
    // per CTA does not fit the grid; WBX_CIRC_SLOTS caps the count
    uint32_t slots = std::max(1u, std::min(batch, static_cast<uint32_t>(num_sms) / P.g0));
    if (batch > slots && multi_m(P, num_sms, batch) > 1) slots = batch;
    if (const char* e = std::getenv("WBX_CIRC_SLOTS")) slots = std::max(1u, std::min(slots, static_cast<uint32_t>(std::atoi(e))));
    return slots;
}


// tracking work (doubles): q [K+1][NB], r and s [K][NB], decoupled sums [2][K][nwd], e0 [2][nwd]
uint64_t circ_track_doubles(const CircPlan& P, int K, int num_sms) {
    const uint64_t NB = P.g0, nwd = static_cast<uint64_t>(num_sms - static_cast<int>(NB)) *
                                    static_cast<uint64_t>(fista_kernel_for(P.g0, P.nCo).warps);
    const uint64_t Kp = static_cast<uint64_t>(K > 0 ? K : 0);
    return (Kp + 1) * NB + 2 * Kp * NB + 2 * Kp * nwd + 2 * nwd + 16;
}

void circ_fista_launch(wbx_ctx* ctx, const CircPlan& P, const CircProblem& pr, const double2* gram, double2* T,
                       unsigned* counter, cudaStream_t st) {
    CircFistaArgs a{};
    const bool track = pr.track_work != nullptr;
    a.x0_full = pr.x0_full;
    a.w_full = pr.w_full;
    a.p_full = pr.p_full;
    a.x_full = pr.x_full;
    a.isC = pr.isC;
    a.n = P.n;
    a.beta64 = pr.beta64;
    a.lambda = pr.lambda;
    a.K = pr.K;
    a.out = pr.out;
    a.gram = gram;
    a.hidx = P.hidx.p;
    a.corb = P.orb.p;
    a.rorb = P.rorb.p;
    a.eoff = P.eoff.p;
    a.eh = P.eh.p;
    a.eval = P.eval.p;
    a.tw = P.tw0.p;
    a.T1 = T;
    a.T2 = T + static_cast<uint64_t>(P.nCo) * P.NG;
    a.counter = counter;
    a.g = P.g0;
    a.lg = static_cast<uint32_t>(__builtin_ctz(P.g0));
    a.nRo = P.nRo;
    a.nCo = P.nCo;
    a.NB = P.g0;
    a.nimg = pr.nimg;
    {  // the staged exchange layout (untracked launches of circ_fista_kernel); WBX_CIRC_STAGED=0: off
        const char* e = std::getenv("WBX_CIRC_STAGED");
        a.staged = !(e && std::string(e) == "0");
    }
    const uint32_t mimg = pr.nimg > 1 ? multi_m(P, ctx->num_sms, pr.nimg) : 1;  // images per CTA
    if (pr.nimg < 1 || mimg == 0 || (track && pr.nimg != 1) || (pr.nimg == 1 && P.g0 >= static_cast<uint32_t>(ctx->num_sms)))
        fail(WBX_BAD_SPEC, "spectral FISTA: images per launch exceed the grid");
    a.diag_skip_decoupled = std::getenv("WBX_CIRC_DIAG") && std::string(std::getenv("WBX_CIRC_DIAG")) == "nodec";
    const FistaKernel k = mimg > 1 ? multi_kernel_for(P.g0, P.nCo, mimg) : fista_kernel_for(P.g0, P.nCo, track);
    if (!k.fn) fail(WBX_BAD_SPEC, "spectral FISTA: unsupported group size");
    a.outw = const_cast<double*>(pr.out);
    if (track) {
        const uint64_t NB = P.g0, nwd = static_cast<uint64_t>(ctx->num_sms - static_cast<int>(NB)) * k.warps;
        const uint64_t Kp = static_cast<uint64_t>(pr.K > 0 ? pr.K : 0);
        a.nwd = static_cast<uint32_t>(nwd);
        a.q_part = pr.track_work;
        a.r_part = a.q_part + (Kp + 1) * NB;
        a.s_part = a.r_part + Kp * NB;
        a.dec_reg = a.s_part + Kp * NB;
        a.dec_sup = a.dec_reg + Kp * nwd;
        a.e0_part = a.dec_sup + Kp * nwd;
        WBX_CUDA(cudaMemsetAsync(a.dec_reg, 0, 2 * Kp * nwd * sizeof(double), st));
    }
#if WBX_CIRC_PROF
    static unsigned long long* prof = nullptr;
    if (!prof) WBX_CUDA(cudaMalloc(&prof, 16 * sizeof(unsigned long long)));
    WBX_CUDA(cudaMemsetAsync(prof, 0, 16 * sizeof(unsigned long long), st));
    a.prof = prof;
#endif
    WBX_CUDA(cudaMemsetAsync(counter, 0, 32u * pr.nimg * sizeof(unsigned), st));
    void* params[] = {&a};
    // one CTA per SM: a single image's launch runs g spectral CTAs and, on the other SMs, its
    // decoupled coordinates; a batch launch runs nimg x g spectral CTAs after the decoupled
    // coordinates of its images in their own launch
    uint32_t grid = static_cast<uint32_t>(ctx->num_sms);
    if (pr.nimg > 1) {
        circ_decoupled_kernel<<<8 * ctx->num_sms, 256, 0, st>>>(pr.x0_full, pr.x_full, pr.w_full, pr.p_full, pr.isC, P.n,
                                                              pr.nimg, pr.beta64, pr.lambda, pr.K, pr.out);
        count_launch(ctx);
        grid = pr.nimg / mimg * P.g0;
    }
    WBX_CUDA(cudaLaunchCooperativeKernel(k.fn, dim3(grid), dim3(32 * k.warps), params, k.smem, st));
    count_launch(ctx);
    WBX_CUDA(cudaGetLastError());
    if (track) {
        circ_energy_kernel<<<pr.K + 1, 256, 0, st>>>(a.q_part, a.r_part, a.s_part, a.dec_reg, a.dec_sup, a.e0_part,
                                                      a.NB, a.nwd, pr.lambda, pr.energies, pr.supports,
                                                      const_cast<double*>(pr.out));
        circ_energy_check_kernel<<<1, 32, 0, st>>>(pr.energies, pr.K, const_cast<double*>(pr.out));
        count_launch(ctx, 2);
        WBX_CUDA(cudaGetLastError());
    }
#if WBX_CIRC_PROF
    unsigned long long h[16];
    WBX_CUDA(cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaStreamSynchronize(st));
    std::fprintf(stderr, "circ_fista cycles per iteration (CTA 0):");
    for (int i = 0; i < 7; ++i) std::fprintf(stderr, " %d:%.0f", i, static_cast<double>(h[i]) / std::max(1, pr.K));
    std::fprintf(stderr, "\n");
#endif
}

void circ_tau_launch(wbx_ctx* ctx, const CircPlan& P, const double* isp_dev, double step_safety, double* work,
                     double2* gram, double* out, cudaStream_t st, cudaStream_t aux, cudaEvent_t ev_fork,
                     cudaEvent_t ev_join) {
    const uint32_t nh = static_cast<uint32_t>(P.h_fhalf.size());
    double* norm_part = work;
    double2* t1 = reinterpret_cast<double2*>(work + kCircNormBlocks);
    double2* vh = t1 + static_cast<uint64_t>(P.nCo) * P.NG;
    double* tri = reinterpret_cast<double*>(vh + static_cast<uint64_t>(P.nCo) * P.NG);
    double* mom_m = tri + static_cast<uint64_t>(2 * kCircMaxCo + 2) * nh;
    int* mom_e = reinterpret_cast<int*>(mom_m + static_cast<uint64_t>(kCircMoments) * nh);
    double* S = reinterpret_cast<double*>(mom_e) + (static_cast<uint64_t>(kCircMoments) * nh + 1) / 2;
    int* X = reinterpret_cast<int*>(S + kCircMoments);
    // G_f (operator only) on the aux stream, beside |v0|^2 and v0's transform (start vector only)
    WBX_CUDA(cudaEventRecord(ev_fork, st));
    WBX_CUDA(cudaStreamWaitEvent(aux, ev_fork, 0));
    circ_gram_launch(ctx, P, gram, aux);
    WBX_CUDA(cudaEventRecord(ev_join, aux));
    circ_norm_kernel<<<kCircNormBlocks, 256, 0, st>>>(P.n, norm_part);
    const unsigned th1 = std::min<uint32_t>(1024, ((P.g1 + 31) / 32) * 32);
    circ_dft1_kernel<<<dim3(P.g0, P.nCo), th1, P.g1 * sizeof(double), st>>>(P.orb.p, P.g0, P.g1, P.tw1.p, t1);
    const unsigned th0 = std::min<uint32_t>(1024, ((P.g0 + 31) / 32) * 32);
    circ_dft0_kernel<<<dim3(P.g1, P.nCo), th0, P.g0 * sizeof(double2), st>>>(P.nCo, P.g0, P.g1, P.tw0.p, t1, vh);
    WBX_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
    circ_lanczos_kernel<<<(nh + 2 * kCircWarps - 1) / (2 * kCircWarps), kCircWarps * 32, 0, st>>>(
        nh, P.fhalf.p, P.nCo, gram, isp_dev, vh, tri);
    const unsigned pb = (nh + 31) / 32;  // one warp per SM: the steps are a dependent chain
    if (P.nCo <= 4)
        circ_power_kernel<4><<<pb, 32, 0, st>>>(nh, tri, mom_m, mom_e);
    else if (P.nCo <= 8)
        circ_power_kernel<8><<<pb, 32, 0, st>>>(nh, tri, mom_m, mom_e);
    else if (P.nCo <= 12)
        circ_power_kernel<12><<<pb, 32, 0, st>>>(nh, tri, mom_m, mom_e);
    else
        circ_power_kernel<16><<<pb, 32, 0, st>>>(nh, tri, mom_m, mom_e);
    unsigned* done = reinterpret_cast<unsigned*>(X + kCircMoments);
    circ_reduce_kernel<<<kCircMoments, 256, 0, st>>>(nh, mom_m, mom_e, S, X, done, P.NG, norm_part, kCircNormBlocks,
                                                     step_safety, out);
    count_launch(ctx, 6);  // + circ_gram_kernel
    WBX_CUDA(cudaGetLastError());
}

}  // namespace wbx

extern "C" int wbx_diag_circ_info(const wbx_op* op, uint32_t ndim, const uint64_t* dims, uint32_t J, uint32_t* info,
                                  char* why, uint64_t why_len) {
    try {
        if (!op || !dims || !info) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_diag_circ_info");
        std::vector<wbx_band> bands;
        wbx::make_layout(ndim, dims, J, bands);
        auto p = wbx::circ_analyze(op, ndim, dims, J, bands);
        std::string w;
        wbx::circ_plan_ok(*p, &w, info);
        if (why && why_len) std::snprintf(why, why_len, "%s", w.c_str());
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}
