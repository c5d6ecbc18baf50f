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
//   circ_norm_kernel     |v0|^2 over all n (one log per Box-Muller pair; block partials)
//   circ_dft1/0_kernel   v^ on the column orbits (separable DFT, twiddle tables)
//   circ_lanczos_kernel  half a warp per frequency: M^_f from the representative rows (staged in
//                        shared memory); Lanczos with full reorthogonalisation -> the real
//                        tridiagonal T_f (<= nCo steps, exact: the Krylov space is the block's)
//   circ_power_kernel    one thread per frequency: the 201 power steps on T_f (5 fma per row
//                        instead of a dense complex matvec), exact power-of-two rescaling, the
//                        402 moments
//   circ_reduce_kernel   per moment, the sum over frequencies with a common exponent (fixed order)
//   circ_final_kernel    lambda_it for every it in parallel, the reference's stopping rule, tau
#include <cmath>
#include <cstring>
#include <string>

#include "internal.hpp"
#include "rng.cuh"
#include "wbx_diag.h"

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
    bool uploaded = false;
    DevBuf<uint32_t> fhalf;
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

// Half a warp per frequency of the half spectrum (f and -f have conjugate blocks and
// transforms, so equal moments: weight 2; self-conjugate frequencies weight 1), two
// frequencies per warp. Lane i < nCo of a half owns row / component i. Every frequency's
// control flow is the same (the representative rows do not depend on f), so the halves do
// not diverge except at a Lanczos breakdown (per-half flags).
//   1. Theta^_f row by row (lane j: column orbit j), M^_f = D Theta^_f^H Theta^_f D (lane i: row i)
//   2. Lanczos on M^_f from v^_f with full reorthogonalisation (classical Gram-Schmidt, twice):
//      the real tridiagonal T_f (k <= nCo) with v^H M^p v = |v|^2 e1^T T^p e1 for every p;
//      written as {alpha[16], beta[16], |v|^2 (weight folded in), k}
__global__ void __launch_bounds__(kCircWarps * 32) circ_lanczos_kernel(
    uint32_t nhalf, const uint32_t* __restrict__ fhalf, uint32_t g1, uint32_t g0, uint32_t nRo, uint32_t nCo,
    const uint32_t* __restrict__ eoff, const uint32_t* __restrict__ eh, const double* __restrict__ eval,
    const double2* __restrict__ tw0, const double2* __restrict__ tw1, const double* __restrict__ isp,
    const double2* __restrict__ vh, double* __restrict__ tri, uint32_t nent) {
    // the representative rows and twiddles, staged once per block (dynamic shared memory)
    extern __shared__ double2 circ_smem[];
    double2* s_tw0 = circ_smem;
    double2* s_tw1 = s_tw0 + g0;
    double* s_val = reinterpret_cast<double*>(s_tw1 + g1);
    uint32_t* s_eh = reinterpret_cast<uint32_t*>(s_val + nent);
    uint32_t* s_eoff = s_eh + nent;
    for (uint32_t i = threadIdx.x; i < g0; i += blockDim.x) s_tw0[i] = tw0[i];
    for (uint32_t i = threadIdx.x; i < g1; i += blockDim.x) s_tw1[i] = tw1[i];
    for (uint32_t i = threadIdx.x; i < nent; i += blockDim.x) {
        s_val[i] = eval[i];
        s_eh[i] = eh[i];
    }
    for (uint32_t i = threadIdx.x; i <= nRo * nCo; i += blockDim.x) s_eoff[i] = eoff[i];
    __syncthreads();
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
    const uint32_t f0 = f / g1, f1 = f % g1;
    const uint32_t m0 = (g0 & (g0 - 1)) == 0 ? g0 - 1 : 0, m1 = (g1 & (g1 - 1)) == 0 ? g1 - 1 : 0;
    const int nc = static_cast<int>(nCo);
    const bool own = li < nc;
    auto half_sum = [](double v) {  // sum over the 16 lanes of this half (identical in every lane)
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };

    // 1. M^_f
    double2 acc[kCircMaxCo];
#pragma unroll
    for (int j = 0; j < kCircMaxCo; ++j) acc[j] = make_double2(0.0, 0.0);
    for (uint32_t r = 0; r < nRo; ++r) {
        if (own) {
            double re = 0.0, im = 0.0;
            for (uint32_t e = s_eoff[r * nCo + li]; e < s_eoff[r * nCo + li + 1]; ++e) {
                const uint32_t h = s_eh[e];
                const uint32_t a0 = f0 * (h >> 16), a1 = f1 * (h & 0xffffu);
                const double2 ph = cmul(s_tw0[m0 ? (a0 & m0) : a0 % g0], s_tw1[m1 ? (a1 & m1) : a1 % g1]);
                re = fma(s_val[e], ph.x, re);
                im = fma(s_val[e], ph.y, im);
            }
            vec[slot][li] = make_double2(re, im);
        }
        __syncwarp();
        if (own) {
            const double2 a = vec[slot][li];  // conj(a) * b
#pragma unroll
            for (int j = 0; j < kCircMaxCo; ++j) {
                if (j < nc) {
                    const double2 b = vec[slot][j];
                    acc[j].x = fma(a.x, b.x, fma(a.y, b.y, acc[j].x));
                    acc[j].y = fma(a.x, b.y, fma(-a.y, b.x, acc[j].y));
                }
            }
        }
        __syncwarp();
    }
    double fro = 0.0;
    if (own) {
        const double di = isp[li];
#pragma unroll
        for (int j = 0; j < kCircMaxCo; ++j) {
            if (j < nc) {
                const double s = di * isp[j];
                const double2 m = make_double2(acc[j].x * s, acc[j].y * s);
                Ms[slot][li][j] = m;
                fro = fma(m.x, m.x, fma(m.y, m.y, fro));
            }
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
__global__ void __launch_bounds__(256) circ_reduce_kernel(uint32_t nhalf, const double* __restrict__ mom_m,
                                                          const int* __restrict__ mom_e, double* S, int* X) {
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
    if (t == 0) {
        S[p] = rs[0];
        X[p] = x == INT_MIN ? 0 : x;
    }
}

// lambda_it for every it from the moments, the reference's stopping rule, tau
__global__ void __launch_bounds__(256) circ_final_kernel(uint32_t NG, const double* __restrict__ Sg,
                                                         const int* __restrict__ Xg, const double* norm_part,
                                                         int norm_blocks, double step_safety, double* out) {
    __shared__ double S[kCircMoments];
    __shared__ int X[kCircMoments];
    __shared__ double lam[200];
    __shared__ int first_stop;
    __shared__ double nv2;
    const int t = threadIdx.x;
    if (t == 0) first_stop = 1 << 30;
    for (int p = t; p < kCircMoments; p += 256) {
        S[p] = Sg[p];
        X[p] = Xg[p];
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
    if (eoff.size() * 4 + P->h_eval.size() * 12 + (g0 + g1) * 16 > 40u * 1024u)
        return no("representative rows too long for shared memory");
    P->h_eoff = std::move(eoff);
    // overflow safety of 4 unnormalised power steps: |M^_f| <= (sum |val|)^2 max(P^-1) is
    // checked per solver (circ_check_p)
    for (uint64_t f0 = 0; f0 < g0; ++f0)  // one of every conjugate pair {f, -f}, weight 2
        for (uint64_t f1 = 0; f1 < g1; ++f1) {
            const uint64_t f = f0 * g1 + f1, fc = ((g0 - f0) % g0) * g1 + (g1 - f1) % g1;
            if (f <= fc) P->h_fhalf.push_back(static_cast<uint32_t>(f << 1 | (f < fc ? 1u : 0u)));
        }
    for (uint64_t k = 0; k < g0; ++k) P->h_tw0.push_back(twiddle(k, g0));
    for (uint64_t k = 0; k < g1; ++k) P->h_tw1.push_back(twiddle(k, g1));
    P->ok = true;
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
    WBX_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(circ_lanczos_kernel),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
    WBX_CUDA(cudaStreamSynchronize(st));
    P.uploaded = true;
}

// Work buffers of one solver's estimate (double-sized units)
uint64_t circ_work_doubles(const CircPlan& P) {
    const uint64_t nh = P.h_fhalf.size();
    return kCircNormBlocks + 4ull * P.nCo * P.NG /* t1, vh */ + (2 * kCircMaxCo + 2) * nh /* T_f */ +
           kCircMoments * nh /* mom_m */ +
           (kCircMoments * nh + 1) / 2 /* mom_e */ + kCircMoments /* S */ + (kCircMoments + 1) / 2 /* X */ + 16;
}

// Enqueue the estimate; writes out[OUT_TAU], out[OUT_TAU_ITERS], out[OUT_LAMBDA_MAX], out[OUT_TAU_STEPS].
void circ_tau_launch(wbx_ctx* ctx, const CircPlan& P, const double* isp_dev, double step_safety, double* work,
                     double* out, cudaStream_t st) {
    const uint32_t nh = static_cast<uint32_t>(P.h_fhalf.size());
    double* norm_part = work;
    double2* t1 = reinterpret_cast<double2*>(work + kCircNormBlocks);
    double2* vh = t1 + static_cast<uint64_t>(P.nCo) * P.NG;
    double* tri = reinterpret_cast<double*>(vh + static_cast<uint64_t>(P.nCo) * P.NG);
    double* mom_m = tri + static_cast<uint64_t>(2 * kCircMaxCo + 2) * nh;
    int* mom_e = reinterpret_cast<int*>(mom_m + static_cast<uint64_t>(kCircMoments) * nh);
    double* S = reinterpret_cast<double*>(mom_e) + (static_cast<uint64_t>(kCircMoments) * nh + 1) / 2;
    int* X = reinterpret_cast<int*>(S + kCircMoments);
    circ_norm_kernel<<<kCircNormBlocks, 256, 0, st>>>(P.n, norm_part);
    const unsigned th1 = std::min<uint32_t>(1024, ((P.g1 + 31) / 32) * 32);
    circ_dft1_kernel<<<dim3(P.g0, P.nCo), th1, P.g1 * sizeof(double), st>>>(P.orb.p, P.g0, P.g1, P.tw1.p, t1);
    const unsigned th0 = std::min<uint32_t>(1024, ((P.g0 + 31) / 32) * 32);
    circ_dft0_kernel<<<dim3(P.g1, P.nCo), th0, P.g0 * sizeof(double2), st>>>(P.nCo, P.g0, P.g1, P.tw0.p, t1, vh);
    const uint32_t nent = static_cast<uint32_t>(P.h_eval.size());
    const size_t lz_smem = (P.g0 + P.g1) * sizeof(double2) + nent * (sizeof(double) + sizeof(uint32_t)) +
                           (P.nRo * P.nCo + 1) * sizeof(uint32_t);
    circ_lanczos_kernel<<<(nh + 2 * kCircWarps - 1) / (2 * kCircWarps), kCircWarps * 32, lz_smem, st>>>(
        nh, P.fhalf.p, P.g1, P.g0, P.nRo, P.nCo, P.eoff.p, P.eh.p, P.eval.p, P.tw0.p, P.tw1.p, isp_dev, vh, tri, nent);
    const unsigned pb = (nh + 31) / 32;  // one warp per SM: the steps are a dependent chain
    if (P.nCo <= 4)
        circ_power_kernel<4><<<pb, 32, 0, st>>>(nh, tri, mom_m, mom_e);
    else if (P.nCo <= 8)
        circ_power_kernel<8><<<pb, 32, 0, st>>>(nh, tri, mom_m, mom_e);
    else if (P.nCo <= 12)
        circ_power_kernel<12><<<pb, 32, 0, st>>>(nh, tri, mom_m, mom_e);
    else
        circ_power_kernel<16><<<pb, 32, 0, st>>>(nh, tri, mom_m, mom_e);
    circ_reduce_kernel<<<kCircMoments, 256, 0, st>>>(nh, mom_m, mom_e, S, X);
    circ_final_kernel<<<1, 256, 0, st>>>(P.NG, S, X, norm_part, kCircNormBlocks, step_safety, out);
    count_launch(ctx, 7);
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
