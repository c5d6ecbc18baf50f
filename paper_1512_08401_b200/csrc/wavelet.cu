// Periodic orthogonal 2-D (and 1-D) Mallat DWT on the device, fp64.
//
// Replaces the reference's analyze/synthesize (`proj/src/wavelet.cpp:118-228,254-260`).
// The arithmetic is the reference's, term for term: every tap is an explicit
// __dmul_rn/__dadd_rn (no FMA contraction, like the reference's x86-64 build), the
// analysis sums run i = 0..l-1 from 0.0 (dwt_line, :86-100) and the synthesis is the
// gather form of idwt_line's scatter-add (:103-115) visiting (k ascending, i ascending)
// exactly as the scatter does, so results are BITWISE equal to the reference.
//
// Data layout: the input image is row-major (dims[0] rows). Forward level t runs a
// rows pass (filter along dim 1) into a scratch plane, then a columns pass that writes
// the three detail subbands STRAIGHT into the band-contiguous coefficient vector
// (make_layout's order, wavelet.cpp:53-66) and the LL quadrant into a compact buffer
// for the next level; at the last level LL lands in band 0. That fuses gather_bands
// (:198-212) into the transform. The inverse mirrors it (scatter_bands fused).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "internal.hpp"

namespace wbx {

namespace {

// Published orthonormal lowpass tables (sum h = sqrt 2, sum h^2 = 1); identical
// decimal literals to the reference tables (wavelet_filters.cpp:14-83), so the doubles
// are identical. Highpass is the quadrature mirror g[i] = (-1)^i h[l-1-i] (:137-142).
const double kHaar[] = {0.70710678118654757, 0.70710678118654757};
const double kDb[11][20] = {
    {},
    {},
    {0.48296291314453416, 0.83651630373780794, 0.22414386804201339, -0.12940952255126037},
    {0.33267055295008263, 0.80689150931109255, 0.45987750211849154, -0.13501102001025458,
     -0.085441273882026658, 0.035226291885709533},
    {0.23037781330889651, 0.71484657055291567, 0.63088076792985892, -0.027983769416859854,
     -0.18703481171909309, 0.030841381835560764, 0.032883011666885197, -0.010597401785069032},
    {0.16010239797419293, 0.60382926979718965, 0.72430852843777294, 0.13842814590132074,
     -0.24229488706638203, -0.032244869584638375, 0.077571493840045719, -0.0062414902127982744,
     -0.012580751999081999, 0.0033357252854737712},
    {0.11154074335010947, 0.49462389039845306, 0.75113390802109536, 0.31525035170919763,
     -0.22626469396543983, -0.12976686756726194, 0.097501605587323043, 0.027522865530305727,
     -0.03158203931748603, 0.00055384220116149613, 0.0047772575109455108,
     -0.0010773010853084796},
    {0.077852054085009184, 0.39653931948191729, 0.72913209084623509, 0.46978228740519312,
     -0.14390600392856498, -0.22403618499387498, 0.071309219266830259, 0.080612609151083078,
     -0.038029936935014413, -0.016574541630666881, 0.01255099855609984, 0.00042957797292136651,
     -0.0018016407040474908, 0.00035371379997452024},
    {0.054415842243104008, 0.31287159091429995, 0.67563073629728976, 0.58535468365420673,
     -0.015829105256349306, -0.28401554296154691, 0.00047248457391328279, 0.12874742662047847,
     -0.017369301001807547, -0.044088253930794755, 0.013981027917398282, 0.0087460940474057766,
     -0.0048703529934515741, -0.00039174037337694705, 0.00067544940645056933,
     -0.00011747678412476953},
    {0.038077947363878345, 0.24383467461259034, 0.60482312369011115, 0.65728807805130052,
     0.13319738582500756, -0.29327378327917492, -0.096840783222976456, 0.14854074933810638,
     0.03072568147933338, -0.067632829061329974, 0.00025094711483145197, 0.022361662123679096,
     -0.0047232047577513972, -0.0042815036824634303, 0.0018476468830562265,
     0.00023038576352319597, -0.00025196318894271012, 3.9347320316271603e-05},
    {0.026670057900555554, 0.1881768000776915, 0.52720118893172563, 0.68845903945360354,
     0.28117234366057747, -0.24984642432731538, -0.19594627437737705, 0.12736934033579325,
     0.093057364603572348, -0.071394147166397082, -0.029457536821875813, 0.033212674059341002,
     0.0036065535669561697, -0.010733175483330575, 0.0013953517470529011, 0.0019924052951850561,
     -0.00068585669495971162, -0.00011646685512928545, 9.3588670320069592e-05,
     -1.3264202894521244e-05},
};
const double kSym[9][16] = {
    {}, {}, {}, {},
    {0.032223100604051466, -0.012603967262031304, -0.099219543576633526, 0.29785779560530606,
     0.8037387518051321, 0.49761866763277501, -0.029635527646002493, -0.075765714789502212},
    {0.027333068344998768, 0.029519490925706261, -0.039134249302313844, 0.19939753397685558,
     0.72340769040404074, 0.63397896345679206, 0.016602105764510849, -0.17532808990805623,
     -0.021101834024689042, 0.019538882735249827},
    {0.015404109327044824, 0.0034907120842221626, -0.11799011114852002, -0.048311742585698057,
     0.49105594192797375, 0.78764114102865102, 0.33792942172816581, -0.072637522786376585,
     -0.021060292512370848, 0.044724901770781388, 0.0017677118642540077,
     -0.0078007083250323803},
    {0.012015419283549189, 0.017213376300804502, -0.064908003547188481, -0.064131289807385819,
     0.3602184609062602, 0.78192159329172817, 0.48361091568226772, -0.056804476889666972,
     -0.1010109208684203, 0.044742349468352378, 0.020464207577546033, -0.018126605131338461,
     -0.0032832978474668108, 0.0022918339540537714},
    {0.0018899503327676891, -0.00030292051472413309, -0.014952258337062199,
     0.0038087520138944896, 0.04913717967373029, -0.027219029917103486, -0.051945838107881802,
     0.36444189483617895, 0.777185751699628, 0.48135965125905339, -0.061273359067811076,
     -0.14329423835127267, 0.0076074873249766086, 0.031695087811525989,
     -0.00054213233180001072, -0.0033824159510050028},
};

// Filter taps passed by value (kernel parameter bank) so concurrent bases never race.
struct Taps {
    double lo[20];
    double hi[20];
    int l;
};

Taps taps_of(const wbx_basis* b) {
    Taps t{};
    std::memcpy(t.lo, b->lo, sizeof t.lo);
    std::memcpy(t.hi, b->hi, sizeof t.hi);
    t.l = static_cast<int>(b->len);
    return t;
}

__device__ __forceinline__ double fma_free(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));
}

// ---------------------------------------------------------------- forward
// dwt_line on every row of an m0 x m1 block: dst[r][k] = lowpass, dst[r][m1/2+k] = highpass.
// A block computes kThreads outputs of one row from a shared-memory copy of the 2 kThreads +
// l - 2 inputs they read (one coalesced load per input instead of l/2 strided ones); the sum
// over taps is the reference's order, so the result is bitwise the same.
__global__ void fwd_rows_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                                int64_t ldd, int m0, int m1, Taps f, int64_t zs) {
    extern __shared__ double sh[];
    src += blockIdx.z * zs;  // image blockIdx.z of a batch (images zs doubles apart in every buffer)
    dst += blockIdx.z * zs;
    const int half = m1 >> 1;
    const int k0 = blockIdx.x * blockDim.x;
    const int r = blockIdx.y;
    if (r >= m0) return;
    const double* row = src + static_cast<int64_t>(r) * lds;
    const int nin = 2 * static_cast<int>(blockDim.x) + f.l - 2;
    for (int t = threadIdx.x; t < nin; t += blockDim.x) {
        int idx = 2 * k0 + t;
        if (idx >= m1) idx %= m1;
        sh[t] = row[idx];
    }
    __syncthreads();
    const int k = k0 + threadIdx.x;
    if (k >= half) return;
    const double* w = sh + 2 * threadIdx.x;
    double a = 0.0, d = 0.0;
    for (int i = 0; i < f.l; ++i) {
        const double s = w[i];
        a = fma_free(a, f.lo[i], s);
        d = fma_free(d, f.hi[i], s);
    }
    dst[static_cast<int64_t>(r) * ldd + k] = a;
    dst[static_cast<int64_t>(r) * ldd + half + k] = d;
}

// dwt_line on every column of the rows-pass output, writing subbands directly.
// Quadrant (row-high e0, col-high e1) -> band orientation e = 2*e0 + e1. A block computes
// kColsOut outputs down kThreads columns from a shared-memory tile of the 2 kColsOut + l - 2
// input rows they read (each input row loaded once per block instead of l/2 times); tap
// order as the reference's (bitwise).
constexpr int kColsOut = 8;
__global__ void fwd_cols_kernel(const double* __restrict__ src, int64_t lds, int m0, int m1, Taps f,
                                double* __restrict__ ll, double* __restrict__ b1,
                                double* __restrict__ b2, double* __restrict__ b3, int64_t zs) {
    extern __shared__ double sh[];
    src += blockIdx.z * zs;
    ll += blockIdx.z * zs;
    b1 += blockIdx.z * zs;
    b2 += blockIdx.z * zs;
    b3 += blockIdx.z * zs;
    const int h0 = m0 >> 1, h1 = m1 >> 1;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int k0 = blockIdx.y * kColsOut;
    const int nrows = 2 * kColsOut + f.l - 2;
    if (c >= m1) return;  // no block-wide barrier below: each thread reads its own column
    for (int t = 0; t < nrows; ++t) {  // all rows in flight (asynchronous copies)
        int idx = 2 * k0 + t;
        if (idx >= m0) idx %= m0;
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sh + t * blockDim.x + threadIdx.x));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src + static_cast<int64_t>(idx) * lds + c)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    for (int kk = 0; kk < kColsOut; ++kk) {
        const int k = k0 + kk;
        if (k >= h0) break;
        double a = 0.0, d = 0.0;
        for (int i = 0; i < f.l; ++i) {
            const double s = sh[(2 * kk + i) * blockDim.x + threadIdx.x];
            a = fma_free(a, f.lo[i], s);
            d = fma_free(d, f.hi[i], s);
        }
        if (c < h1) {
            ll[static_cast<int64_t>(k) * h1 + c] = a;
            b2[static_cast<int64_t>(k) * h1 + c] = d;
        } else {
            b1[static_cast<int64_t>(k) * h1 + (c - h1)] = a;
            b3[static_cast<int64_t>(k) * h1 + (c - h1)] = d;
        }
    }
}

// 1-D level: lowpass -> ll, highpass -> band.
__global__ void fwd_line_kernel(const double* __restrict__ src, int m, Taps f, double* __restrict__ ll,
                                double* __restrict__ hb) {
    const int half = m >> 1;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= half) return;
    double a = 0.0, d = 0.0;
    for (int i = 0; i < f.l; ++i) {
        const double s = src[(2 * k + i) % m];
        a = fma_free(a, f.lo[i], s);
        d = fma_free(d, f.hi[i], s);
    }
    ll[k] = a;
    hb[k] = d;
}

// ---------------------------------------------------------------- inverse
// Output j of idwt_line over a line of length m (half h): sum over (k asc, i asc) with
// (2k+i) mod m == j of (a_k*lo[i] + d_k*hi[i]), starting from 0.0 — the exact order in
// which the reference's scatter-add (wavelet.cpp:108-114) reaches out[j].
template <typename LoadA, typename LoadD>
__device__ __forceinline__ double idwt_point(int j, int m, const Taps& f, LoadA A, LoadD D) {
    const int h = m >> 1;
    double out = 0.0;
    if (m >= f.l) {
        // non-wrapped k in [max(0, ceil((j-l+1)/2)), floor(j/2)]
        int kmin = j - f.l + 1;
        kmin = kmin <= 0 ? 0 : (kmin + 1) >> 1;
        const int kmax = j >> 1;
        for (int k = kmin; k <= kmax; ++k) {
            const int i = j - 2 * k;
            out = __dadd_rn(out, __dadd_rn(__dmul_rn(A(k), f.lo[i]), __dmul_rn(D(k), f.hi[i])));
        }
        // wrapped k (2k > j) with j + m - 2k in [0, l)
        int wmin = j + m - f.l + 1;
        wmin = (wmin + 1) >> 1;
        if (wmin < kmax + 1) wmin = kmax + 1;
        int wmax = (j + m) >> 1;
        if (wmax > h - 1) wmax = h - 1;
        for (int k = wmin; k <= wmax; ++k) {
            const int i = j + m - 2 * k;
            out = __dadd_rn(out, __dadd_rn(__dmul_rn(A(k), f.lo[i]), __dmul_rn(D(k), f.hi[i])));
        }
    } else {
        for (int k = 0; k < h; ++k) {
            int i = (j - 2 * k) % m;
            if (i < 0) i += m;
            for (; i < f.l; i += m)
                out = __dadd_rn(out,
                                __dadd_rn(__dmul_rn(A(k), f.lo[i]), __dmul_rn(D(k), f.hi[i])));
        }
    }
    return out;
}

// Columns pass of inverse level: V[j][c], c < h1 from (LL, band2), else (band1, band3).
__global__ void inv_cols_kernel(const double* __restrict__ ll, const double* __restrict__ b1,
                                const double* __restrict__ b2, const double* __restrict__ b3,
                                int m0, int m1, Taps f, double* __restrict__ dst, int64_t zs) {
    ll += blockIdx.z * zs;
    b1 += blockIdx.z * zs;
    b2 += blockIdx.z * zs;
    b3 += blockIdx.z * zs;
    dst += blockIdx.z * zs;
    const int h1 = m1 >> 1;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (c >= m1 || j >= m0) return;
    const double* pa = c < h1 ? ll + c : b1 + (c - h1);
    const double* pd = c < h1 ? b2 + c : b3 + (c - h1);
    const double v = idwt_point(
        j, m0, f, [&](int k) { return pa[static_cast<int64_t>(k) * h1]; },
        [&](int k) { return pd[static_cast<int64_t>(k) * h1]; });
    dst[static_cast<int64_t>(j) * m1 + c] = v;
}

// Rows pass of inverse level: out[j][x] from V[j][0:h1] (lowpass) and V[j][h1:m1].
// clamp: the deblur's final std::clamp(v, 0, 1) (waveblur.cpp:297) fused into the last level
__global__ void inv_rows_kernel(const double* __restrict__ src, int m0, int m1, Taps f,
                                double* __restrict__ dst, int64_t ldd, int clamp, int64_t zs) {
    src += blockIdx.z * zs;
    dst += blockIdx.z * zs;
    const int h1 = m1 >> 1;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (x >= m1 || j >= m0) return;
    const double* row = src + static_cast<int64_t>(j) * m1;
    double v = idwt_point(
        x, m1, f, [&](int k) { return row[k]; }, [&](int k) { return row[h1 + k]; });
    if (clamp) v = fmin(fmax(v, 0.0), 1.0);
    dst[static_cast<int64_t>(j) * ldd + x] = v;
}

__global__ void inv_line_kernel(const double* __restrict__ ll, const double* __restrict__ hb, int m,
                                Taps f, double* __restrict__ dst, int clamp) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    double v = idwt_point(j, m, f, [&](int k) { return ll[k]; }, [&](int k) { return hb[k]; });
    if (clamp) v = fmin(fmax(v, 0.0), 1.0);
    dst[j] = v;
}

inline int band_index(const wbx_basis* b, uint32_t t, uint32_t e) {
    const int per_level = b->ndim == 2 ? 3 : 1;
    return 1 + static_cast<int>(b->J - t) * per_level + static_cast<int>(e) - 1;
}

constexpr int kThreads = 128;

}  // namespace

void make_filters(uint32_t family, uint32_t order, double* lo, double* hi, uint32_t* len) {
    const double* t = nullptr;
    uint32_t l = 0;
    switch (family) {
        case WBX_HAAR:
            if (order != 1) fail(WBX_UNSUPPORTED_FILTER, "Haar has order 1 only");
            t = kHaar;
            l = 2;
            break;
        case WBX_DAUBECHIES:
            if (order < 2 || order > 10) fail(WBX_UNSUPPORTED_FILTER, "Daubechies order must be in 2..10");
            t = kDb[order];
            l = 2 * order;
            break;
        case WBX_SYMMLET:
            if (order < 4 || order > 8) fail(WBX_UNSUPPORTED_FILTER, "Symmlet order must be in 4..8");
            t = kSym[order];
            l = 2 * order;
            break;
        default:
            fail(WBX_UNSUPPORTED_FILTER, "unknown filter family");
    }
    // orthonormality check (wavelet_filters.cpp:85-97)
    double s2 = 0.0;
    for (uint32_t i = 0; i < l; ++i) s2 += t[i] * t[i];
    if (std::abs(s2 - 1.0) > 1e-12) fail(WBX_UNSUPPORTED_FILTER, "filter table failed unit-norm check");
    for (uint32_t k = 1; 2 * k < l; ++k) {
        double s = 0.0;
        for (uint32_t i = 0; i + 2 * k < l; ++i) s += t[i] * t[i + 2 * k];
        if (std::abs(s) > 1e-12)
            fail(WBX_UNSUPPORTED_FILTER, "filter table failed shift-orthogonality check");
    }
    for (uint32_t i = 0; i < l; ++i) {
        lo[i] = t[i];
        hi[i] = ((i % 2 == 0) ? 1.0 : -1.0) * t[l - 1 - i];
    }
    *len = l;
}

void make_layout(uint32_t ndim, const uint64_t* dims, uint32_t J, std::vector<wbx_band>& bands) {
    if (ndim < 1 || ndim > 2) fail(WBX_SHAPE_MISMATCH, "layout needs 1 or 2 dims");
    uint64_t mind = dims[0];
    for (uint32_t k = 0; k < ndim; ++k) {
        if (dims[k] == 0 || (dims[k] & (dims[k] - 1)) != 0)
            fail(WBX_SHAPE_MISMATCH, "side lengths must be powers of 2");
        mind = std::min(mind, dims[k]);
    }
    if (J < 1 || J >= 63 || (uint64_t{1} << J) > mind)
        fail(WBX_SHAPE_MISMATCH, "decomposition depth too deep for these dims");
    bands.clear();
    uint64_t off = 0;
    auto push = [&](uint32_t t, uint32_t e) {
        wbx_band b{};
        b.level = t;
        b.orientation = e;
        b.shape[0] = dims[0] >> t;
        b.shape[1] = ndim == 2 ? (dims[1] >> t) : 1;
        b.offset = off;
        off += b.shape[0] * b.shape[1];
        bands.push_back(b);
    };
    push(J, 0);
    for (uint32_t t = J; t >= 1; --t)
        for (uint32_t e = 1; e < (1u << ndim); ++e) push(t, e);
}

void analyze_dev(wbx_basis* b, const double* u, double* x, cudaStream_t s) {
    analyze_dev_n(b, u, x, 1, b->work_a.p, b->work_b.p, s);
}

// nimg images back to back (n doubles apart in u, x and both n-per-image work buffers): each
// 2-D level pass is one launch over all images (blockIdx.z); 1-D bases run image by image
void analyze_dev_n(wbx_basis* b, const double* u, double* x, uint32_t nimg, double* work_a, double* work_b,
                   cudaStream_t s) {
    const Taps f = taps_of(b);
    double* tmp = work_a;
    double* llbuf = work_b;
    const int64_t zs = static_cast<int64_t>(b->n);
    if (b->ndim == 1 && nimg > 1) {
        for (uint32_t i = 0; i < nimg; ++i) analyze_dev_n(b, u + i * b->n, x + i * b->n, 1, work_a, work_b, s);
        return;
    }
    if (b->ndim == 1) {
        const double* src = u;
        for (uint32_t t = 0; t < b->J; ++t) {
            const int m = static_cast<int>(b->dims[0] >> t);
            const bool last = t + 1 == b->J;
            double* ll = last ? x + b->bands[0].offset : (t % 2 == 0 ? llbuf : tmp);
            double* hb = x + b->bands[band_index(b, t + 1, 1)].offset;
            fwd_line_kernel<<<(m / 2 + kThreads - 1) / kThreads, kThreads, 0, s>>>(src, m, f, ll, hb);
            count_launch(b->ctx);
            src = ll;
        }
    } else {
        const double* src = u;
        int64_t lds = static_cast<int64_t>(b->dims[1]);
        for (uint32_t t = 0; t < b->J; ++t) {
            const int m0 = static_cast<int>(b->dims[0] >> t), m1 = static_cast<int>(b->dims[1] >> t);
            const bool last = t + 1 == b->J;
            dim3 g1((m1 / 2 + kThreads - 1) / kThreads, m0, nimg);
            fwd_rows_kernel<<<g1, kThreads, (2 * kThreads + f.l) * sizeof(double), s>>>(src, lds, tmp, m1, m0, m1, f, zs);
            double* ll = last ? x + b->bands[0].offset : llbuf;
            double* b1 = x + b->bands[band_index(b, t + 1, 1)].offset;
            double* b2 = x + b->bands[band_index(b, t + 1, 2)].offset;
            double* b3 = x + b->bands[band_index(b, t + 1, 3)].offset;
            dim3 g2((m1 + kThreads - 1) / kThreads, (m0 / 2 + kColsOut - 1) / kColsOut, nimg);
            fwd_cols_kernel<<<g2, kThreads, (2 * kColsOut + f.l) * kThreads * sizeof(double), s>>>(tmp, m1, m0, m1, f, ll,
                                                                                                  b1, b2, b3, zs);
            count_launch(b->ctx, 2);
            src = ll;
            lds = m1 / 2;
        }
    }
    WBX_CUDA(cudaGetLastError());
}

void synthesize_dev(wbx_basis* b, const double* x, double* u, cudaStream_t s, int clamp) {
    synthesize_dev_n(b, x, u, 1, b->work_a.p, b->work_b.p, s, clamp);
}

void synthesize_dev_n(wbx_basis* b, const double* x, double* u, uint32_t nimg, double* work_a, double* work_b,
                      cudaStream_t s, int clamp) {
    const Taps f = taps_of(b);
    double* tmp = work_a;
    double* llbufs[2] = {work_b, work_b + b->n / 2};
    const int64_t zs = static_cast<int64_t>(b->n);
    if (b->ndim == 1 && nimg > 1) {
        for (uint32_t i = 0; i < nimg; ++i) synthesize_dev_n(b, x + i * b->n, u + i * b->n, 1, work_a, work_b, s, clamp);
        return;
    }
    if (b->ndim == 1) {
        const double* ll = x + b->bands[0].offset;
        int which = 0;
        for (uint32_t t = b->J; t >= 1; --t) {
            const int m = static_cast<int>(b->dims[0] >> (t - 1));
            const double* hb = x + b->bands[band_index(b, t, 1)].offset;
            double* dst = t == 1 ? u : llbufs[which];
            inv_line_kernel<<<(m + kThreads - 1) / kThreads, kThreads, 0, s>>>(ll, hb, m, f, dst, t == 1 ? clamp : 0);
            count_launch(b->ctx);
            ll = dst;
            which ^= 1;
        }
    } else {
        const double* ll = x + b->bands[0].offset;
        int which = 0;
        for (uint32_t t = b->J; t >= 1; --t) {
            const int m0 = static_cast<int>(b->dims[0] >> (t - 1)), m1 = static_cast<int>(b->dims[1] >> (t - 1));
            const double* b1 = x + b->bands[band_index(b, t, 1)].offset;
            const double* b2 = x + b->bands[band_index(b, t, 2)].offset;
            const double* b3 = x + b->bands[band_index(b, t, 3)].offset;
            dim3 g((m1 + kThreads - 1) / kThreads, m0, nimg);
            inv_cols_kernel<<<g, kThreads, 0, s>>>(ll, b1, b2, b3, m0, m1, f, tmp, zs);
            double* dst = t == 1 ? u : llbufs[which];
            inv_rows_kernel<<<g, kThreads, 0, s>>>(tmp, m0, m1, f, dst, m1, t == 1 ? clamp : 0, zs);
            count_launch(b->ctx, 2);
            ll = dst;
            which ^= 1;
        }
    }
    WBX_CUDA(cudaGetLastError());
}

}  // namespace wbx
