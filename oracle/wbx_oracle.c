/* oracle/wbx_oracle.c — TEST INFRASTRUCTURE ONLY (see wbx_oracle.h).
 *
 * fp64 serial restatement of the reference hot path. Statement order follows the
 * cited reference lines exactly; compile with -ffp-contract=off.
 */
#define _GNU_SOURCE
#include "wbx_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ filters
 * Published orthonormal lowpass tables (sum h = sqrt 2, sum h^2 = 1), the same
 * decimal literals as the reference tables (wavelet_filters.cpp:14-83) so the
 * parsed doubles are identical. Highpass g[i] = (-1)^i h[l-1-i] (:137-142). */
static const double kHaar[2] = {0.70710678118654757, 0.70710678118654757};
static const double kDb2[4] = {0.48296291314453416, 0.83651630373780794, 0.22414386804201339,
                               -0.12940952255126037};
static const double kDb3[6] = {0.33267055295008263, 0.80689150931109255, 0.45987750211849154,
                               -0.13501102001025458, -0.085441273882026658, 0.035226291885709533};
static const double kDb4[8] = {0.23037781330889651,   0.71484657055291567,  0.63088076792985892,
                               -0.027983769416859854, -0.18703481171909309, 0.030841381835560764,
                               0.032883011666885197,  -0.010597401785069032};
static const double kDb5[10] = {0.16010239797419293,   0.60382926979718965,
                                0.72430852843777294,   0.13842814590132074,
                                -0.24229488706638203,  -0.032244869584638375,
                                0.077571493840045719,  -0.0062414902127982744,
                                -0.012580751999081999, 0.0033357252854737712};
static const double kDb6[12] = {0.11154074335010947,    0.49462389039845306,
                                0.75113390802109536,    0.31525035170919763,
                                -0.22626469396543983,   -0.12976686756726194,
                                0.097501605587323043,   0.027522865530305727,
                                -0.03158203931748603,   0.00055384220116149613,
                                0.0047772575109455108,  -0.0010773010853084796};
static const double kDb7[14] = {0.077852054085009184,  0.39653931948191729,
                                0.72913209084623509,   0.46978228740519312,
                                -0.14390600392856498,  -0.22403618499387498,
                                0.071309219266830259,  0.080612609151083078,
                                -0.038029936935014413, -0.016574541630666881,
                                0.01255099855609984,   0.00042957797292136651,
                                -0.0018016407040474908, 0.00035371379997452024};
static const double kDb8[16] = {0.054415842243104008,   0.31287159091429995,
                                0.67563073629728976,    0.58535468365420673,
                                -0.015829105256349306,  -0.28401554296154691,
                                0.00047248457391328279, 0.12874742662047847,
                                -0.017369301001807547,  -0.044088253930794755,
                                0.013981027917398282,   0.0087460940474057766,
                                -0.0048703529934515741, -0.00039174037337694705,
                                0.00067544940645056933, -0.00011747678412476953};
static const double kDb9[18] = {0.038077947363878345,   0.24383467461259034,
                                0.60482312369011115,    0.65728807805130052,
                                0.13319738582500756,    -0.29327378327917492,
                                -0.096840783222976456,  0.14854074933810638,
                                0.03072568147933338,    -0.067632829061329974,
                                0.00025094711483145197, 0.022361662123679096,
                                -0.0047232047577513972, -0.0042815036824634303,
                                0.0018476468830562265,  0.00023038576352319597,
                                -0.00025196318894271012, 3.9347320316271603e-05};
static const double kDb10[20] = {0.026670057900555554,   0.1881768000776915,
                                 0.52720118893172563,    0.68845903945360354,
                                 0.28117234366057747,    -0.24984642432731538,
                                 -0.19594627437737705,   0.12736934033579325,
                                 0.093057364603572348,   -0.071394147166397082,
                                 -0.029457536821875813,  0.033212674059341002,
                                 0.0036065535669561697,  -0.010733175483330575,
                                 0.0013953517470529011,  0.0019924052951850561,
                                 -0.00068585669495971162, -0.00011646685512928545,
                                 9.3588670320069592e-05, -1.3264202894521244e-05};
static const double kSym4[8] = {0.032223100604051466, -0.012603967262031304,
                                -0.099219543576633526, 0.29785779560530606,
                                0.8037387518051321,    0.49761866763277501,
                                -0.029635527646002493, -0.075765714789502212};
static const double kSym5[10] = {0.027333068344998768,  0.029519490925706261,
                                 -0.039134249302313844, 0.19939753397685558,
                                 0.72340769040404074,   0.63397896345679206,
                                 0.016602105764510849,  -0.17532808990805623,
                                 -0.021101834024689042, 0.019538882735249827};
static const double kSym6[12] = {0.015404109327044824,  0.0034907120842221626,
                                 -0.11799011114852002,  -0.048311742585698057,
                                 0.49105594192797375,   0.78764114102865102,
                                 0.33792942172816581,   -0.072637522786376585,
                                 -0.021060292512370848, 0.044724901770781388,
                                 0.0017677118642540077, -0.0078007083250323803};
static const double kSym7[14] = {0.012015419283549189,   0.017213376300804502,
                                 -0.064908003547188481,  -0.064131289807385819,
                                 0.3602184609062602,     0.78192159329172817,
                                 0.48361091568226772,    -0.056804476889666972,
                                 -0.1010109208684203,    0.044742349468352378,
                                 0.020464207577546033,   -0.018126605131338461,
                                 -0.0032832978474668108, 0.0022918339540537714};
static const double kSym8[16] = {0.0018899503327676891,  -0.00030292051472413309,
                                 -0.014952258337062199,  0.0038087520138944896,
                                 0.04913717967373029,    -0.027219029917103486,
                                 -0.051945838107881802,  0.36444189483617895,
                                 0.777185751699628,      0.48135965125905339,
                                 -0.061273359067811076,  -0.14329423835127267,
                                 0.0076074873249766086,  0.031695087811525989,
                                 -0.00054213233180001072, -0.0033824159510050028};

int wbxo_filters(uint32_t family, uint32_t order, double* lo, double* hi, uint32_t* len) {
    const double* t = NULL;
    uint32_t l = 0;
    if (family == 0) {
        if (order != 1) return WBXO_UNSUPPORTED_FILTER;
        t = kHaar;
        l = 2;
    } else if (family == 1) {
        static const double* const db[11] = {NULL, NULL, kDb2, kDb3, kDb4, kDb5,
                                             kDb6, kDb7, kDb8, kDb9, kDb10};
        if (order < 2 || order > 10) return WBXO_UNSUPPORTED_FILTER;
        t = db[order];
        l = 2 * order;
    } else if (family == 2) {
        static const double* const sy[9] = {NULL, NULL, NULL, NULL, kSym4, kSym5, kSym6, kSym7, kSym8};
        if (order < 4 || order > 8) return WBXO_UNSUPPORTED_FILTER;
        t = sy[order];
        l = 2 * order;
    } else {
        return WBXO_UNSUPPORTED_FILTER;
    }
    for (uint32_t i = 0; i < l; ++i) {
        lo[i] = t[i];
        hi[i] = ((i % 2 == 0) ? 1.0 : -1.0) * t[l - 1 - i];
    }
    *len = l;
    return WBXO_OK;
}

/* ------------------------------------------------------------------ layout */
static int is_pow2(uint64_t n) { return n > 0 && (n & (n - 1)) == 0; }

int wbxo_layout(uint32_t ndim, const uint64_t* dims, uint32_t J, wbxo_band* bands) {
    if (ndim < 1 || ndim > 2) return -WBXO_SHAPE;
    uint64_t mind = dims[0];
    for (uint32_t k = 0; k < ndim; ++k) {
        if (!is_pow2(dims[k])) return -WBXO_SHAPE;
        if (dims[k] < mind) mind = dims[k];
    }
    if (J < 1 || ((uint64_t)1 << J) > mind) return -WBXO_SHAPE;
    int nb = 0;
    uint64_t off = 0;
    const uint32_t ne = 1u << ndim;
    for (int pass = 0; pass < 2; ++pass) {
        /* pass 0: approximation (J,0); pass 1: details t = J..1, e = 1..2^d-1 */
        for (uint32_t t = J; t >= 1; --t) {
            for (uint32_t e = (pass == 0 ? 0u : 1u); e < (pass == 0 ? 1u : ne); ++e) {
                wbxo_band* b = &bands[nb++];
                b->level = t;
                b->orientation = e;
                b->shape[0] = dims[0] >> t;
                b->shape[1] = ndim == 2 ? (dims[1] >> t) : 1;
                b->offset = off;
                off += b->shape[0] * b->shape[1];
            }
            if (pass == 0) break;
        }
    }
    return nb;
}

/* ------------------------------------------------------------------ DWT */
/* dwt_line (wavelet.cpp:86-100) */
static void dwt_line(const double* in, size_t stride, size_t n, const double* lo, const double* hi,
                     size_t l, double* out) {
    const size_t half = n / 2;
    for (size_t k = 0; k < half; ++k) {
        double a = 0.0, d = 0.0;
        for (size_t i = 0; i < l; ++i) {
            double s = in[((2 * k + i) % n) * stride];
            a += lo[i] * s;
            d += hi[i] * s;
        }
        out[k] = a;
        out[half + k] = d;
    }
}

/* idwt_line (wavelet.cpp:103-115) */
static void idwt_line(const double* in, size_t stride, size_t n, const double* lo,
                      const double* hi, size_t l, double* out) {
    const size_t half = n / 2;
    for (size_t j = 0; j < n; ++j) out[j] = 0.0;
    for (size_t k = 0; k < half; ++k) {
        const double a = in[k * stride];
        const double d = in[(half + k) * stride];
        for (size_t i = 0; i < l; ++i) out[(2 * k + i) % n] += a * lo[i] + d * hi[i];
    }
}

static size_t mallat_origin(const wbxo_band* b, uint32_t ndim, const uint64_t* dims) {
    if (ndim == 1) return (b->orientation & 1u) ? (size_t)(dims[0] >> b->level) : 0;
    size_t r0 = ((b->orientation >> 1) & 1u) ? (size_t)(dims[0] >> b->level) : 0;
    size_t c0 = (b->orientation & 1u) ? (size_t)(dims[1] >> b->level) : 0;
    return r0 * (size_t)dims[1] + c0;
}

int wbxo_analyze(uint32_t ndim, const uint64_t* dims, uint32_t J, const double* lo,
                 const double* hi, uint32_t len, const double* u, double* x) {
    wbxo_band bands[64];
    int nb = wbxo_layout(ndim, dims, J, bands);
    if (nb < 0) return -nb;
    const size_t n0 = dims[0], n1 = ndim == 2 ? dims[1] : 1, N = n0 * n1;
    double* w = malloc(N * sizeof(double));
    double* tmp = malloc((n0 > n1 ? n0 : n1) * sizeof(double));
    memcpy(w, u, N * sizeof(double));
    if (ndim == 1) { /* wavelet.cpp:120-129 */
        for (uint32_t t = 0; t < J; ++t) {
            const size_t nt = n0 >> t;
            dwt_line(w, 1, nt, lo, hi, len, tmp);
            memcpy(w, tmp, nt * sizeof(double));
        }
    } else { /* wavelet.cpp:130-148: rows then columns per level */
        const size_t cols = n1;
        for (uint32_t t = 0; t < J; ++t) {
            const size_t m0 = n0 >> t, m1 = n1 >> t;
            for (size_t r = 0; r < m0; ++r) {
                double* row = w + r * cols;
                dwt_line(row, 1, m1, lo, hi, len, tmp);
                memcpy(row, tmp, m1 * sizeof(double));
            }
            for (size_t c = 0; c < m1; ++c) {
                double* col = w + c;
                dwt_line(col, cols, m0, lo, hi, len, tmp);
                for (size_t r = 0; r < m0; ++r) col[r * cols] = tmp[r];
            }
        }
    }
    /* gather_bands (wavelet.cpp:198-212) */
    for (int bi = 0; bi < nb; ++bi) {
        const wbxo_band* b = &bands[bi];
        const size_t o = mallat_origin(b, ndim, dims);
        for (size_t r = 0; r < b->shape[0]; ++r)
            for (size_t c = 0; c < b->shape[1]; ++c)
                x[b->offset + r * b->shape[1] + c] = w[o + r * n1 + c];
    }
    free(w);
    free(tmp);
    return WBXO_OK;
}

int wbxo_synthesize(uint32_t ndim, const uint64_t* dims, uint32_t J, const double* lo,
                    const double* hi, uint32_t len, const double* x, double* u) {
    wbxo_band bands[64];
    int nb = wbxo_layout(ndim, dims, J, bands);
    if (nb < 0) return -nb;
    const size_t n0 = dims[0], n1 = ndim == 2 ? dims[1] : 1, N = n0 * n1;
    double* w = u;
    double* tmp = malloc((n0 > n1 ? n0 : n1) * sizeof(double));
    /* scatter_bands (wavelet.cpp:214-228) */
    for (size_t i = 0; i < N; ++i) w[i] = 0.0;
    for (int bi = 0; bi < nb; ++bi) {
        const wbxo_band* b = &bands[bi];
        const size_t o = mallat_origin(b, ndim, dims);
        for (size_t r = 0; r < b->shape[0]; ++r)
            for (size_t c = 0; c < b->shape[1]; ++c)
                w[o + r * n1 + c] = x[b->offset + r * b->shape[1] + c];
    }
    if (ndim == 1) { /* wavelet.cpp:153-162 */
        for (uint32_t t = J; t >= 1; --t) {
            const size_t nt = n0 >> (t - 1);
            idwt_line(w, 1, nt, lo, hi, len, tmp);
            memcpy(w, tmp, nt * sizeof(double));
        }
    } else { /* wavelet.cpp:163-181: columns then rows, coarse to fine */
        const size_t cols = n1;
        for (uint32_t t = J; t >= 1; --t) {
            const size_t m0 = n0 >> (t - 1), m1 = n1 >> (t - 1);
            for (size_t c = 0; c < m1; ++c) {
                double* col = w + c;
                idwt_line(col, cols, m0, lo, hi, len, tmp);
                for (size_t r = 0; r < m0; ++r) col[r * cols] = tmp[r];
            }
            for (size_t r = 0; r < m0; ++r) {
                double* row = w + r * cols;
                idwt_line(row, 1, m1, lo, hi, len, tmp);
                memcpy(row, tmp, m1 * sizeof(double));
            }
        }
    }
    free(tmp);
    return WBXO_OK;
}

/* ------------------------------------------------------------------ SpMV */
void wbxo_spmv(const wbxo_csr* op, const double* x, double* y) {
    for (uint64_t r = 0; r < op->n; ++r) {
        double s = 0.0;
        for (uint64_t k = op->row_offsets[r]; k < op->row_offsets[r + 1]; ++k)
            s += op->values[k] * x[op->col_indices[k]];
        y[r] = s;
    }
}

void wbxo_transpose(const wbxo_csr* op, uint64_t* t_off, uint32_t* t_idx, double* t_val) {
    const uint64_t n = op->n;
    const uint64_t nnz = op->row_offsets[n];
    for (uint64_t i = 0; i <= n; ++i) t_off[i] = 0;
    for (uint64_t k = 0; k < nnz; ++k) ++t_off[op->col_indices[k] + 1];
    for (uint64_t i = 0; i < n; ++i) t_off[i + 1] += t_off[i];
    uint64_t* cursor = malloc((n ? n : 1) * sizeof(uint64_t));
    memcpy(cursor, t_off, n * sizeof(uint64_t));
    for (uint64_t r = 0; r < n; ++r) {
        for (uint64_t k = op->row_offsets[r]; k < op->row_offsets[r + 1]; ++k) {
            uint64_t pos = cursor[op->col_indices[k]]++;
            t_idx[pos] = (uint32_t)r;
            t_val[pos] = op->values[k];
        }
    }
    free(cursor);
}

/* ------------------------------------------------------------------ solver pieces */
void wbxo_prox(uint64_t n, const double* z0, double tau, const double* w, double lambda,
               const double* p, double* z) {
    for (uint64_t i = 0; i < n; ++i) {
        double thr = tau * lambda * w[i] / p[i];
        double a = fabs(z0[i]) - thr;
        z[i] = a > 0.0 ? (z0[i] > 0.0 ? a : -a) : 0.0;
    }
}

void wbxo_scale_weights(uint32_t nb, const wbxo_band* bands, uint32_t J, double* w) {
    for (uint32_t b = 0; b < nb; ++b) {
        double v = bands[b].orientation == 0 ? (double)J : (double)bands[b].level;
        const uint64_t cnt = bands[b].shape[0] * bands[b].shape[1];
        for (uint64_t i = 0; i < cnt; ++i) w[bands[b].offset + i] = v;
    }
}

static double dot(const double* a, const double* b, uint64_t n) {
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

double wbxo_energy(const wbxo_csr* op, const double* x, const double* x0, const double* w,
                   double lambda, uint64_t n) {
    double* r = malloc(n * sizeof(double));
    wbxo_spmv(op, x, r);
    double quad = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        double d = r[i] - x0[i];
        quad += d * d;
    }
    double reg = 0.0;
    for (uint64_t i = 0; i < n; ++i) reg += w[i] * fabs(x[i]);
    free(r);
    return 0.5 * quad + lambda * reg;
}

/* ------------------------------------------------------------------ CounterRng */
uint64_t wbxo_rng_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (i + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static double u01(uint64_t v) { return ((double)(v >> 11) + 0.5) * 0x1p-53; }

void wbxo_rng_uniforms(uint64_t seed, uint64_t n, double* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = u01(wbxo_rng_at(seed, i));
}

void wbxo_rng_normals(uint64_t seed, uint64_t n, double* out) {
    /* next_normal (rng.hpp:30-43): draws 2m, 2m+1 -> cos for element 2m, sin for 2m+1 */
    for (uint64_t m = 0; 2 * m < n; ++m) {
        double u1 = u01(wbxo_rng_at(seed, 2 * m));
        double u2 = u01(wbxo_rng_at(seed, 2 * m + 1));
        double r = sqrt(-2.0 * log(u1));
        double a = 2.0 * M_PI * u2;
        out[2 * m] = r * cos(a);
        if (2 * m + 1 < n) out[2 * m + 1] = r * sin(a);
    }
}

/* ------------------------------------------------------------------ estimate_step */
double wbxo_estimate_step(const wbxo_csr* op, const wbxo_csr* tr, const double* p,
                          double step_safety, uint32_t* iters_out) {
    const uint64_t n = op->n;
    double* isp = malloc(n * sizeof(double));
    double* v = malloc(n * sizeof(double));
    double* w = malloc(n * sizeof(double));
    double* t = malloc(n * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) isp[i] = 1.0 / sqrt(p[i]);
    wbxo_rng_normals(0x5eedULL, n, v);
    double nv = sqrt(dot(v, v, n));
    for (uint64_t i = 0; i < n; ++i) v[i] /= nv;
    double lambda_prev = 0.0;
    double result = -1.0;
    uint32_t it_done = 0;
    for (int it = 0; it < 200; ++it) {
        for (uint64_t i = 0; i < n; ++i) w[i] = isp[i] * v[i];
        wbxo_spmv(op, w, t);
        wbxo_spmv(tr, t, w);
        for (uint64_t i = 0; i < n; ++i) w[i] *= isp[i];
        double lambda = dot(v, w, n);
        double nw = sqrt(dot(w, w, n));
        it_done = (uint32_t)it + 1;
        if (nw == 0.0) {
            result = 1.0;
            break;
        }
        for (uint64_t i = 0; i < n; ++i) v[i] = w[i] / nw;
        if (it > 0 && fabs(lambda - lambda_prev) <= 1e-6 * fabs(lambda)) {
            lambda_prev = lambda;
            break;
        }
        lambda_prev = lambda;
    }
    if (result < 0.0) result = lambda_prev <= 0.0 ? 1.0 : 1.0 / (lambda_prev * step_safety);
    if (iters_out) *iters_out = it_done;
    free(isp);
    free(v);
    free(w);
    free(t);
    return result;
}

/* ------------------------------------------------------------------ run_pgd */
static int pgd_loop(const wbxo_csr* op, const wbxo_csr* tr, const double* x0, const double* w,
                    double lambda, const double* p, double tau, uint64_t max_iters,
                    double stop_gap, double ref_energy, int zero_momentum, int accelerate,
                    double* x_final, double* energies, uint64_t* iters_used) {
    const uint64_t n = op->n;
    double* xp = malloc(n * sizeof(double));
    double* y = malloc(n * sizeof(double));
    double* r = malloc(n * sizeof(double));
    double* g = malloc(n * sizeof(double));
    double* xn = malloc(n * sizeof(double));
    memcpy(xp, x0, n * sizeof(double));
    memcpy(y, x0, n * sizeof(double));
    memcpy(x_final, x0, n * sizeof(double));
    int status = WBXO_OK;
    uint64_t used = 0;
    for (uint64_t k = 1; k <= max_iters; ++k) {
        wbxo_spmv(op, y, r);
        for (uint64_t i = 0; i < n; ++i) r[i] -= x0[i];
        wbxo_spmv(tr, r, g);
        for (uint64_t i = 0; i < n; ++i) xn[i] = y[i] - tau * g[i] / p[i]; /* z0 */
        wbxo_prox(n, xn, tau, w, lambda, p, xn);
        double e = 0.0;
        if (energies || isfinite(ref_energy)) {
            e = wbxo_energy(op, xn, x0, w, lambda, n);
            if (!isfinite(e)) {
                status = WBXO_NONFINITE;
                break;
            }
            if (energies) energies[k - 1] = e;
        }
        double beta = 0.0;
        if (accelerate && !zero_momentum) beta = ((double)k - 1.0) / ((double)k + 2.0);
        for (uint64_t i = 0; i < n; ++i) y[i] = xn[i] + beta * (xn[i] - xp[i]);
        memcpy(xp, xn, n * sizeof(double));
        memcpy(x_final, xn, n * sizeof(double));
        used = k;
        if (isfinite(ref_energy) && e - ref_energy <= stop_gap) break;
    }
    if (iters_used) *iters_used = used;
    free(xp);
    free(y);
    free(r);
    free(g);
    free(xn);
    return status;
}

int wbxo_pgd(const wbxo_csr* op, const wbxo_csr* tr, const double* x0, const double* w,
             double lambda, const double* p, uint64_t max_iters, double rel_energy_tol,
             double step_safety, double ref_energy, int zero_momentum, int accelerate,
             double* x_final, double* energies, uint64_t* iters_used, double* tau_out,
             double* initial_energy) {
    const double tau = wbxo_estimate_step(op, tr, p, step_safety, NULL);
    const double e0 = wbxo_energy(op, x0, x0, w, lambda, op->n);
    if (tau_out) *tau_out = tau;
    if (initial_energy) *initial_energy = e0;
    return pgd_loop(op, tr, x0, w, lambda, p, tau, max_iters, rel_energy_tol * e0, ref_energy,
                    zero_momentum, accelerate, x_final, energies, iters_used);
}

int wbxo_pgd_tau(const wbxo_csr* op, const wbxo_csr* tr, const double* x0, const double* w,
                 double lambda, const double* p, double tau, uint64_t max_iters,
                 int zero_momentum, int accelerate, double* x_final) {
    return pgd_loop(op, tr, x0, w, lambda, p, tau, max_iters, 0.0, NAN, zero_momentum,
                    accelerate, x_final, NULL, NULL);
}

/* ------------------------------------------------------------------ preconditioners */
int wbxo_gram_diagonals(const wbxo_csr* op, uint64_t nnz_cap_factor, double* diagM,
                        double* diagM2) {
    const uint64_t n = op->n, nnz = op->row_offsets[n];
    uint64_t* t_off = malloc((n + 1) * sizeof(uint64_t));
    uint32_t* t_idx = malloc((nnz ? nnz : 1) * sizeof(uint32_t));
    double* t_val = malloc((nnz ? nnz : 1) * sizeof(double));
    wbxo_transpose(op, t_off, t_idx, t_val);
    for (uint64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (uint64_t k = t_off[i]; k < t_off[i + 1]; ++k) s += t_val[k] * t_val[k];
        diagM[i] = s;
    }
    const uint64_t cap = nnz_cap_factor * (nnz > 1 ? nnz : 1);
    uint64_t m_nnz = 0;
    double* acc = calloc(n ? n : 1, sizeof(double));
    uint32_t* touched = malloc((n ? n : 1) * 4 * sizeof(uint32_t));
    uint64_t touched_cap = (n ? n : 1) * 4;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t nt = 0;
        for (uint64_t k = t_off[i]; k < t_off[i + 1]; ++k) {
            const uint32_t row = t_idx[k];
            const double a = t_val[k];
            for (uint64_t j = op->row_offsets[row]; j < op->row_offsets[row + 1]; ++j) {
                const uint32_t col = op->col_indices[j];
                if (acc[col] == 0.0) {
                    if (nt == touched_cap) {
                        touched_cap *= 2;
                        touched = realloc(touched, touched_cap * sizeof(uint32_t));
                    }
                    touched[nt++] = col;
                }
                acc[col] += a * op->values[j];
            }
        }
        double s = 0.0;
        for (uint64_t q = 0; q < nt; ++q) {
            s += acc[touched[q]] * acc[touched[q]];
            acc[touched[q]] = 0.0;
        }
        diagM2[i] = s;
        m_nnz += nt;
    }
    free(acc);
    free(touched);
    free(t_off);
    free(t_idx);
    free(t_val);
    return m_nnz > cap ? WBXO_MEMORY_GUARD : WBXO_OK;
}

int wbxo_spai(const wbxo_csr* op, double* p) {
    const uint64_t n = op->n;
    double* m = malloc((n ? n : 1) * sizeof(double));
    double* m2 = malloc((n ? n : 1) * sizeof(double));
    int st = wbxo_gram_diagonals(op, 50, m, m2);
    if (st == WBXO_OK)
        for (uint64_t i = 0; i < n; ++i) p[i] = m[i] > 0.0 ? m2[i] / m[i] : 1.0;
    free(m);
    free(m2);
    return st;
}

int wbxo_jacobi(const wbxo_csr* op, double eps, double* p) {
    if (eps <= 0.0) return WBXO_BAD_EPSILON;
    const uint64_t n = op->n;
    double* m = malloc((n ? n : 1) * sizeof(double));
    double* m2 = malloc((n ? n : 1) * sizeof(double));
    int st = wbxo_gram_diagonals(op, 50, m, m2);
    if (st == WBXO_OK)
        for (uint64_t i = 0; i < n; ++i) p[i] = m[i] < eps ? eps : m[i]; /* std::max(m, eps) */
    free(m);
    free(m2);
    return st;
}
