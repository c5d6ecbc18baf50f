/* oracle/shim/fftw3.h — TEST INFRASTRUCTURE ONLY (oracle build of the reference).
 *
 * FFTW3 is a third-party dependency of the reference (`proj/src/operators.cpp:9`,
 * `proj/CMakeLists.txt:14-15`) that is absent from this image and not vendored in
 * /root/reference (no version is pinned anywhere in the reference; the system
 * package is implied). The reference uses exactly six entry points of it
 * (`operators.cpp:20-68`): r2c/c2r plans in 1-D and 2-D with FFTW_ESTIMATE,
 * fftw_execute and fftw_destroy_plan. This header restates that published API
 * for power-of-two sizes (the reference only ever builds dyadic grids,
 * `image.hpp:73-78`):
 *   r2c: out[k] = sum_j in[j] exp(-2 pi i j.k / N) over the last axis' n/2+1 bins
 *   c2r: out[j] = sum_k in[k] exp(+2 pi i j.k / N) over the full Hermitian
 *        spectrum — UNNORMALISED, exactly as FFTW (the reference divides by N
 *        itself, `operators.cpp:65-66`).
 * The transform is an iterative radix-2 Cooley-Tukey FFT with directly evaluated
 * twiddles (fftw_shim.cpp). Results agree with FFTW to ~1e-15 relative, not
 * bitwise; every reference tolerance that involves the FFT is >= 1e-12
 * (`test_operators.cpp:110-125,156-169`), and the oracle's Theta_K index set is
 * pinned to THIS build.
 */
#ifndef WBX_ORACLE_FFTW3_SHIM_H
#define WBX_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct wbx_fftw_plan_s* fftw_plan;

#define FFTW_ESTIMATE (1U << 6)
#define FFTW_MEASURE (0U)

fftw_plan fftw_plan_dft_r2c_1d(int n, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_r2c_2d(int n0, int n1, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex* in, double* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r_2d(int n0, int n1, fftw_complex* in, double* out, unsigned flags);
void fftw_execute(const fftw_plan plan);
void fftw_destroy_plan(fftw_plan plan);

#ifdef __cplusplus
}
#endif

#endif
