/* include/wbx.h — C ABI of the B200-native waveblur hot path (libwbx.so).
 *
 * This is the drop-in boundary. The reference (waveblur, C++20, CPU/OpenMP) exposes
 * its hot path as a C++ header API only; every entry point below replaces one of
 * those functions (file:line citations are relative to /root/reference/proj) and
 * keeps its argument meaning and error behaviour. Plain pointers and sizes only.
 *
 *   * Host-pointer entry points take/return the reference's fp64 vectors
 *     (std::vector<double> in the reference) and synchronise before returning.
 *   * `_dev` entry points take device pointers and are asynchronous on the
 *     context's stream (wbx_ctx_stream).
 *   * Every function returns a wbx_status; the message of the last failure on the
 *     calling thread is available from wbx_last_error(). Status codes map 1:1 onto
 *     the reference's exception types (`include/waveblur/image.hpp:10-36`), which the
 *     reference-side binding (integration/wbx_backend.cpp) re-throws.
 *   * A context binds one CUDA device and one stream; calls on one context must be
 *     serialised by the caller (the reference's functions are pure and re-entrant;
 *     use one context per host thread for the same property). Per-call scratch lives
 *     in the calling context, so two contexts may use one operator concurrently.
 *   * Lifetimes: a basis or operator must outlive every solver, shard or exact operator
 *     built on it (they keep pointers to its device layouts, like the reference's
 *     non-owning `WaveletCoeffs.layout` / `DeblurProblem.op`, wavelet.hpp:81-84,
 *     solver.hpp:56); a context must outlive every object created on it.
 */
#ifndef WBX_H
#define WBX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WBX_ABI_VERSION 1

typedef enum {
    WBX_OK = 0,
    WBX_SHAPE_MISMATCH = 1,     /* ShapeMismatch      (image.hpp:10)  */
    WBX_UNSUPPORTED_FILTER = 2, /* UnsupportedFilter  (image.hpp:13)  */
    WBX_BAND_NOT_FOUND = 3,     /* BandNotFound       (image.hpp:16)  */
    WBX_BAD_SPEC = 4,           /* BadSpec            (image.hpp:19)  */
    WBX_TOO_LARGE = 5,          /* TooLarge           (image.hpp:22)  */
    WBX_BAD_EPSILON = 6,        /* BadEpsilon         (image.hpp:25)  */
    WBX_MEMORY_GUARD = 7,       /* MemoryGuard        (image.hpp:28)  */
    WBX_NONFINITE_ENERGY = 8,   /* NonFiniteEnergy    (image.hpp:31)  */
    WBX_IO_ERROR = 9,           /* IoError            (image.hpp:34)  */
    WBX_CUDA_ERROR = 10,        /* device failure (no reference equivalent) */
    WBX_INVALID_ARGUMENT = 11   /* null handle / pointer                    */
} wbx_status;

typedef enum { WBX_HAAR = 0, WBX_DAUBECHIES = 1, WBX_SYMMLET = 2 } wbx_family; /* FilterFamily, wavelet.hpp:12 */
typedef enum { WBX_FP32 = 32, WBX_FP64 = 64 } wbx_precision;

typedef struct wbx_ctx wbx_ctx;     /* device + stream + scratch                        */
typedef struct wbx_basis wbx_basis; /* WaveletBasis (wavelet.hpp:68-74) resident on device */
typedef struct wbx_op wbx_op;       /* SparseThetaOp (solver.hpp:25-38): Theta_K + cached transpose */
typedef struct wbx_solver wbx_solver; /* a prepared preconditioned-FISTA solve (op, P, w, lambda, tau) */

typedef struct {
    uint32_t level, orientation; /* Band (wavelet.hpp:39-52) */
    uint64_t shape[2];           /* shape[1] == 1 for 1-D layouts */
    uint64_t offset;
} wbx_band;

/* SolverConfig (solver.hpp:66-74) + device knobs */
typedef struct {
    uint64_t max_iters;      /* default 500 */
    double rel_energy_tol;   /* default 1e-3 */
    double step_safety;      /* default 1.01 */
    double ref_energy;       /* NaN disables the energy stopping rule */
    int32_t zero_momentum;   /* test hook: beta = 0 */
    int32_t track_support;   /* fill report.support_sizes */
    int32_t track_energy;    /* fill report.energies (forced on when ref_energy is finite) */
    int32_t precision;       /* WBX_FP32 (hot path) or WBX_FP64 (bitwise reference mode) */
    double tau;              /* > 0: use this step instead of estimate_step (e.g. cached) */
} wbx_solver_cfg;

/* SolveReport (solver.hpp:76-84). energies / support_sizes are caller-allocated
 * (length >= max_iters) or NULL. */
typedef struct {
    uint64_t iters_used;
    double initial_energy;
    double wall_time_s;         /* device time of the solve incl. tau, CUDA events */
    double tau;                 /* the step actually used */
    uint32_t tau_iters;         /* power iterations spent (0 when tau was given) */
    double ops_per_pixel_per_iter;
    double* energies;
    uint64_t* support_sizes;
} wbx_report;

typedef struct {
    uint64_t n, nnz;
    uint64_t nonempty_rows, nonempty_cols; /* |R| and |C| of the compacted layouts */
    uint64_t sell_rows_padded, sell_cols_padded;
    uint64_t device_bytes;
    uint64_t bytes_per_iter_fp32;          /* algorithmic HBM bytes of one FISTA iteration */
} wbx_op_info;

/* ---------------------------------------------------------------- context */
const char* wbx_last_error(void);
int wbx_abi_version(void);
int wbx_ctx_create(int device, wbx_ctx** out);
int wbx_ctx_destroy(wbx_ctx* ctx);
void* wbx_ctx_stream(wbx_ctx* ctx); /* cudaStream_t */
int wbx_ctx_synchronize(wbx_ctx* ctx);
/* number of kernels this library launched on ctx since creation (launch accounting) */
uint64_t wbx_ctx_launch_count(const wbx_ctx* ctx);

/* ---------------------------------------------------------------- wavelets */
/* make_filters (wavelet_filters.cpp:110-144); lo/hi must hold 20 doubles */
int wbx_make_filters(uint32_t family, uint32_t order, double* lo, double* hi, uint32_t* length);
/* make_filters(name) (wavelet_filters.cpp:146-161): "haar", "db4", "sym6", "symmlet6" */
int wbx_parse_filter(const char* name, uint32_t* family, uint32_t* order);
/* make_layout (wavelet.cpp:32-70); bands must hold 1 + 3*J entries; returns count */
int wbx_make_layout(uint32_t ndim, const uint64_t* dims, uint32_t J, wbx_band* bands,
                    uint32_t* nbands);
int wbx_basis_create(wbx_ctx* ctx, uint32_t family, uint32_t order, uint32_t ndim,
                     const uint64_t* dims, uint32_t J, wbx_basis** out);
int wbx_basis_destroy(wbx_basis* basis);
/* analyze (wavelet.cpp:254-256): x = Psi^* u; fp64, bitwise equal to the reference */
int wbx_analyze(wbx_ctx* ctx, const wbx_basis* basis, const double* u, double* x);
/* synthesize (wavelet.cpp:258-260): u = Psi x; fp64, bitwise equal to the reference */
int wbx_synthesize(wbx_ctx* ctx, const wbx_basis* basis, const double* x, double* u);
int wbx_analyze_dev(wbx_ctx* ctx, const wbx_basis* basis, const double* u_dev, double* x_dev);
int wbx_synthesize_dev(wbx_ctx* ctx, const wbx_basis* basis, const double* x_dev, double* u_dev);
/* single_wavelet (wavelet.cpp:262-269) */
int wbx_single_wavelet(wbx_ctx* ctx, const wbx_basis* basis, uint32_t level, uint32_t orientation,
                       double* u);

/* ---------------------------------------------------------------- Theta_K */
/* Upload a CSR Theta_K (SparseOperator, theta.hpp:50-60) and build the device layouts
 * (compacted sliced-ELL of Theta and of its transpose, fp32 + fp64 values). Validates
 * like read_operator (theta.cpp:479-488): WBX_SHAPE_MISMATCH on bad offsets/columns. */
int wbx_op_create(wbx_ctx* ctx, uint64_t n, const uint64_t* row_offsets,
                  const uint32_t* col_indices, const double* values, wbx_op** out);
int wbx_op_destroy(wbx_op* op);
int wbx_op_get_info(const wbx_op* op, wbx_op_info* info);
/* spmv / SparseThetaOp::apply (theta.cpp:300-311, solver.cpp:11-13) when transpose == 0;
 * SparseThetaOp::apply_adjoint / spmv_t (solver.cpp:15-17, theta.cpp:344-356) when 1.
 * fp64 with the reference's in-row order: bitwise equal to the reference. */
int wbx_spmv(wbx_ctx* ctx, const wbx_op* op, int transpose, const double* x, double* y);
int wbx_spmv_dev(wbx_ctx* ctx, const wbx_op* op, int transpose, int precision, const void* x_dev,
                 void* y_dev);
/* The SELL kernel of wbx_spmv_dev alone, in the compacted spaces (no gather/scatter/memset):
 * transpose == 0: y[|R|] = Theta[R, C] x[|C|]; 1: y[|C|] = Theta^T[C, R] x[|R|]
 * (|R|, |C| = wbx_op_info.nonempty_rows / nonempty_cols). Same arithmetic as wbx_spmv_dev;
 * used to measure the SpMV against the HBM roofline (tools/spmv_roofline.py). */
int wbx_spmv_compact_dev(wbx_ctx* ctx, const wbx_op* op, int transpose, int precision,
                         const void* x_dev, void* y_dev);
/* Attach the kept generator groups (wbx_theta_expand format) of a stationary Theta_K to its
 * operator; they must expand to the operator's CSR exactly (WBX_BAD_SPEC otherwise). Solvers on
 * the operator may then run the stencil engine (no index stream: every entry of a circulant
 * block is an affine function of its output position; csrc/stencil_engine.cuh). */
int wbx_op_set_generators(wbx_op* op, uint32_t ndim, const uint64_t* dims, uint32_t J, uint64_t n_gens,
                          const uint32_t* blocks, const uint32_t* gen_index, const uint64_t* counts,
                          const double* values);
/* Attach the wavelet layout the operator acts on (SparseOperator::layout, theta.hpp:55; also set
 * by wbx_op_set_generators). Solvers created without a basis (wbx_pgd: the reference's fista() /
 * ista()) use it for the block-Fourier step estimate of translation-invariant operators
 * (csrc/circ_tau.cu). make_layout's errors; WBX_SHAPE_MISMATCH when the sizes differ. */
int wbx_op_set_layout(wbx_op* op, uint32_t ndim, const uint64_t* dims, uint32_t J);
/* write_operator / read_operator (theta.cpp:413-490): the reference's WTHETA01 file, same
 * bytes, same validation (WBX_IO_ERROR with the reference's messages; bad layouts raise what
 * make_layout raises). read: the arrays are allocated by the library (malloc; wbx_free);
 * dims must hold 2 entries. */
int wbx_write_operator(const char* path, uint32_t ndim, const uint64_t* dims, uint32_t J, uint32_t family,
                       uint32_t order, uint64_t n, const uint64_t* row_offsets, const uint32_t* col_indices,
                       const double* values);
int wbx_read_operator(const char* path, uint32_t* ndim, uint64_t* dims, uint32_t* J, uint32_t* family,
                      uint32_t* order, uint64_t* n, uint64_t* nnz, uint64_t** row_offsets,
                      uint32_t** col_indices, double** values);
/* Device-ready operator cache (WBXOP001; no reference counterpart): everything
 * wbx_op_create built (compacted orders, exact fp64 SELL, fp32 layouts of Theta and Theta^T)
 * plus the window layouts solvers built since, and optionally the operator's preconditioner p
 * (n doubles, may be NULL) and step tau (0 = none). wbx_op_load uploads them without
 * recomputing anything; p (n doubles) / has_p / tau may be NULL. */
int wbx_op_save(const wbx_op* op, const char* path, const double* p, double tau);
int wbx_op_load(wbx_ctx* ctx, const char* path, wbx_op** out, double* p, int* has_p, double* tau);
/* The operator's CSR (SparseThetaOp::sparse(), solver.hpp:33): row_offsets n + 1, columns and
 * values nnz (wbx_op_get_info) entries, caller-allocated. */
int wbx_op_get_csr(const wbx_op* op, uint64_t* row_offsets, uint32_t* col_indices, double* values);
/* approx_gradient (theta.cpp:358-365): Theta^T (Theta x - x0) */
int wbx_approx_gradient(wbx_ctx* ctx, const wbx_op* op, const double* x, const double* x0,
                        double* g);
/* Expand a thresholded circulant operator given as kept generator groups (the
 * reference's top-K walk, theta.cpp:236-275, + assemble :180-201) into CSR.
 * gens: n_gens records {block = out*nbands + in, gen_index, count, value}.
 * Call with row_offsets/col_indices/values == NULL to query nnz first. */
int wbx_theta_expand(uint32_t ndim, const uint64_t* dims, uint32_t J, uint64_t n_gens,
                     const uint32_t* blocks, const uint32_t* gen_index, const uint64_t* counts,
                     const double* values, uint64_t* nnz, uint64_t* row_offsets,
                     uint32_t* col_indices, double* out_values);

/* Theta_K construction on the device (build_theta_conv theta.cpp:40-79 + threshold_impl
 * theta.cpp:206-276): the blurred single wavelets of every band (FFT convolution in the
 * oracle build's exact arithmetic, see csrc/theta_gpu.cu), their analyses, the weighted keys
 * |g| * band_weight[in] of every generator entry and the global top-K walk. Output: the kept
 * generator groups in the reference's walk order (wbx_theta_expand input); n_records <=
 * max_records. band_weight[b] is the per-band sigma of threshold_weighted (dyadic_weights:
 * 2^(level - J); all ones for threshold_naive). psf: the kernel image (row-major). */
int wbx_theta_conv_topk(wbx_ctx* ctx, wbx_basis* basis, const double* psf, const double* band_weight, uint64_t K,
                        uint64_t max_records, uint32_t* gen_block, uint32_t* gen_index, uint64_t* gen_count,
                        double* gen_value, uint64_t* n_records);
/* gaussian_kernel + normalize_sum (operators.cpp:100-120, 84-89): the PSF image of
 * generate_psf(GaussianSpec{sigma}) (host). */
int wbx_psf_gaussian(uint32_t ndim, const uint64_t* dims, double sigma, double* kernel);

/* ---------------------------------------------------------------- PSFs, convolution, degrade
 * generate_psf (operators.cpp:298-318; PsfSpec, operators.hpp:15-36): the kernel image on the
 * full grid (centred at index 0, wrap-around, unit mass), same expressions as the reference
 * (bitwise). params by kind: GAUSSIAN {sigma}, SKEWED {sigma}, MOTION {points, sigma1, sigma2,
 * seed} (MotionSpec defaults 5, 8, 1, 0), AIRY {scale}, DEFOCUS {radius}. ctx: needed by MOTION
 * (its Gaussian post-smoothing is a device FFT convolution), may be NULL otherwise.
 * BadSpec on bad parameters, ShapeMismatch on non-dyadic dims (Image::require_dyadic). */
typedef enum {
    WBX_PSF_GAUSSIAN = 0,
    WBX_PSF_SKEWED = 1,
    WBX_PSF_MOTION = 2,
    WBX_PSF_AIRY = 3,
    WBX_PSF_DEFOCUS = 4
} wbx_psf_kind;
int wbx_generate_psf(wbx_ctx* ctx, uint32_t kind, const double* params, uint32_t ndim, const uint64_t* dims,
                     double* kernel);
/* convolve / apply_adjoint (operators.cpp:320-326, convolve_spectral :20-77): circular
 * convolution with the kernel image (adjoint: with h~[i] = h[-i]) through the device FFT, in
 * the oracle build's FFT arithmetic. Host images, synchronous. */
int wbx_convolve(wbx_ctx* ctx, uint32_t ndim, const uint64_t* dims, const double* kernel, const double* u,
                 int adjoint, double* out);
/* add_noise (operators.cpp:344-356): u + sigma * N(0,1), per-index Box-Muller on
 * CounterRng(seed) draws 2i, 2i+1; on the device. degrade (operators.cpp:385-387) =
 * add_noise(convolve(u, psf), noise_sigma, seed). */
int wbx_add_noise(wbx_ctx* ctx, uint64_t n, const double* u, double sigma, uint64_t seed, double* out);
int wbx_degrade(wbx_ctx* ctx, uint32_t ndim, const uint64_t* dims, const double* kernel, const double* u,
                double noise_sigma, uint64_t seed, double* out);

/* Spatially varying Theta_K (BASELINE configs C3/C4; the reference has no 2-D spatially
 * varying operator): column mu = the column of the stationary operator whose
 * Gaussian sigma matches the spatial row of psi_mu, sigma varying linearly from
 * sigma_first_row (image row 0) to sigma_last_row (row H), linearly interpolated between
 * the two bracketing levels of a sigma ladder; the column's index set is the union of the
 * two levels' sets. Levels are given as concatenated generator lists (wbx_theta_expand
 * format) with level_ngens[l] records each. Output arrays are allocated by the library
 * (malloc) and released with wbx_free. */
int wbx_theta_varying(uint32_t ndim, const uint64_t* dims, uint32_t J, uint32_t nlevels,
                      const double* sigmas, const uint64_t* level_ngens, const uint32_t* blocks,
                      const uint32_t* gen_index, const uint64_t* counts, const double* values,
                      double sigma_first_row, double sigma_last_row, uint64_t* nnz,
                      uint64_t** row_offsets, uint32_t** col_indices, double** out_values);
void wbx_free(void* p);

/* ---------------------------------------------------------------- preconditioners */
/* gram_diagonals (precond.cpp:16-67), spai (:79-87), jacobi (:69-77); fp64, bitwise */
int wbx_gram_diagonals(wbx_ctx* ctx, const wbx_op* op, uint64_t nnz_cap_factor, double* diagM,
                       double* diagM2);
int wbx_spai(wbx_ctx* ctx, const wbx_op* op, double* p);
int wbx_jacobi(wbx_ctx* ctx, const wbx_op* op, double eps, double* p);

/* ---------------------------------------------------------------- solver */
/* scale_weights (solver.cpp:33-42) */
int wbx_scale_weights(uint32_t ndim, const uint64_t* dims, uint32_t J, double* w);
/* prox_weighted_l1_P (solver.cpp:57-67), on device, fp64 */
int wbx_prox_l1w(wbx_ctx* ctx, uint64_t n, const double* z0, double tau, const double* w,
                 double lambda, const double* p, double* z);
/* energy (solver.cpp:44-55) */
int wbx_energy(wbx_ctx* ctx, const wbx_op* op, const double* x, const double* x0,
               const double* w, double lambda, double* e);
/* estimate_step (solver.cpp:69-99): fp64 power iteration on the device */
int wbx_estimate_step(wbx_ctx* ctx, const wbx_op* op, const double* p, double step_safety,
                      double* tau, uint32_t* iters);
void wbx_solver_cfg_default(wbx_solver_cfg* cfg);
/* ista / fista (solver.cpp:161-169 -> run_pgd :103-157). x_final: n doubles. */
int wbx_pgd(wbx_ctx* ctx, const wbx_op* op, const double* x0, const double* w, double lambda,
            const double* p, const wbx_solver_cfg* cfg, int accelerate, double* x_final,
            wbx_report* report);

/* ---------------------------------------------------------------- stencil operator
 * Theta_K in circulant-compressed form: the kept generator groups
 * (wbx_theta_expand input) applied directly, y = Theta x or Theta^T x, reading only x and y
 * (no CSR). Row sums in record order (equal to wbx_spmv within rounding). precision:
 * WBX_FP64 (double x, y) or WBX_FP32 (float x, y); device pointers. */
typedef struct wbx_stencil wbx_stencil;
int wbx_stencil_create(wbx_ctx* ctx, uint32_t ndim, const uint64_t* dims, uint32_t J, uint64_t n_gens,
                       const uint32_t* blocks, const uint32_t* gen_index, const uint64_t* counts,
                       const double* values, wbx_stencil** out);
int wbx_stencil_destroy(wbx_stencil* s);
int wbx_stencil_spmv_dev(wbx_stencil* s, int transpose, int precision, const void* x_dev, void* y_dev);

/* ---------------------------------------------------------------- exact FFT operator
 * ExactThetaOp (solver.cpp:21-29): Theta x = analyze(convolve(synthesize(x), psf)), the
 * adjoint with the conjugated kernel spectrum; bitwise the reference's (oracle FFT
 * arithmetic, fft.cuh). estimate_step / run_pgd over it (solver.cpp:69-157): the reference's
 * per-coordinate expressions in fp64, fixed-order reductions. psf: the kernel image. */
typedef struct wbx_exact_op wbx_exact_op;
int wbx_exact_op_create(wbx_ctx* ctx, wbx_basis* basis, const double* psf, wbx_exact_op** out);
int wbx_exact_op_destroy(wbx_exact_op* e);
int wbx_exact_apply(wbx_exact_op* e, int adjoint, const double* x, double* y);
int wbx_exact_apply_dev(wbx_exact_op* e, int adjoint, const double* x_dev, double* y_dev);
int wbx_estimate_step_exact(wbx_exact_op* e, const double* p, double step_safety, double* tau, uint32_t* iters);
int wbx_pgd_exact(wbx_exact_op* e, const double* x0, const double* w, double lambda, const double* p,
                  const wbx_solver_cfg* cfg, int accelerate, double* x_final, wbx_report* report);

/* ---------------------------------------------------------------- prepared deblur (hot path)
 * The unit the bench times: u0 (observed image) -> analyze -> [estimate_step] ->
 * preconditioned FISTA -> synthesize -> restored image (pre-clamp; clamp=1 applies the
 * CLI's [0,1] clamp, waveblur.cpp:296-297). Mirrors cmd_deblur's solve
 * (waveblur.cpp:286-297) with the operator, P, w, lambda bound once. */
int wbx_solver_create(wbx_ctx* ctx, const wbx_op* op, const wbx_basis* basis, const double* p,
                      const double* w, double lambda, const wbx_solver_cfg* cfg,
                      wbx_solver** out);
int wbx_solver_destroy(wbx_solver* s);
/* device pointers (fp64 images, n doubles), async on the ctx stream */
int wbx_deblur_dev(wbx_solver* s, const double* u0_dev, double* u_dev, int clamp);
/* host pointers: H2D copy, deblur, D2H copy, synchronise */
int wbx_deblur(wbx_solver* s, const double* u0, double* u, int clamp, wbx_report* report);
/* Batched deblur (BASELINE config C5): `batch` (1, 4 or 8) independent images share Theta_K,
 * P, w, lambda and tau (estimated once per batch). Images are stored back to back (batch * n
 * doubles) for wbx_deblur / wbx_deblur_dev. Translation-invariant operators run the fp64
 * spectral engine with the whole batch in one launch (up to 4 images per CTA); others stream
 * the operator once per batch (fp32 SpMM). precision = WBX_FP32 (the hot-path setting), no
 * energy tracking, fixed iteration count; every image equals its single-image solve bitwise. */
int wbx_solver_create_batch(wbx_ctx* ctx, const wbx_op* op, const wbx_basis* basis, const double* p,
                            const double* w, double lambda, const wbx_solver_cfg* cfg, int batch,
                            wbx_solver** out);
int wbx_solver_batch(const wbx_solver* s);
/* ---------------------------------------------------------------- row-sharded solve (C4)
 * One image across `world` ranks (one per GPU). Rank `rank` owns a contiguous,
 * nnz-balanced range of the compacted rows of Theta and of Theta^T. Cross-rank vectors live in
 * caller-owned PADDED device buffers (rank q's slice at q * max_range): y (fp32, world*maxC),
 * res (fp32, world*maxR), u (fp64, world*maxC), t (fp64, world*maxR). After each phase the
 * caller all-gathers the owned slice (NCCL all_gather over NVLink, or a copy when emulated).
 * Per FISTA iteration k: phase_a -> all-gather res -> phase_t(k) -> all-gather y.
 * estimate_step (solver.cpp:69-99) stays on the device: bind_power gives the caller-owned
 * fp64 sums buffer [world][2]; power_begin -> all-gather sums -> power_update(first=1) ->
 * 200 x { power_step_a -> all-gather t -> power_step_t -> all-gather sums ->
 * power_update(0) -> all-gather u } -> power_result. Every rank sums the slots in rank
 * order and applies the stopping rule itself; once stopped the remaining enqueued steps are
 * no-ops, so the host never waits inside the loop. A sharded solve is bitwise equal to the
 * single-GPU fp32 solve given the same tau, for any world size. */
typedef struct wbx_shard wbx_shard;
int wbx_shard_create(wbx_ctx* ctx, uint64_t n, const uint64_t* row_offsets, const uint32_t* col_indices,
                     const double* values, uint32_t world, uint32_t rank, wbx_shard** out);
int wbx_shard_destroy(wbx_shard* s);
/* host-only partition plan (what wbx_shard_create uses): rbounds/cbounds[world + 1] */
int wbx_shard_plan(uint64_t n, const uint64_t* row_offsets, const uint32_t* col_indices, uint32_t world,
                   uint64_t* rbounds, uint64_t* cbounds);
/* info8 = {world, rank, row_lo, row_hi, col_lo, col_hi, maxR, maxC} */
int wbx_shard_get_info(const wbx_shard* s, uint64_t* info8);
int wbx_shard_bind(wbx_shard* s, float* y_pad, float* res_pad, double* u_pad, double* t_pad);
int wbx_shard_setup(wbx_shard* s, const double* p, const double* w, double lambda, int max_iters,
                    int accelerate);
int wbx_shard_init(wbx_shard* s, double tau, const double* x0_full_dev, double* x_full_dev);
int wbx_shard_phase_a(wbx_shard* s);
int wbx_shard_phase_t(wbx_shard* s, int k);
int wbx_shard_finalize(wbx_shard* s, double* x_full_dev);
int wbx_shard_bind_power(wbx_shard* s, double* sums_pad);
int wbx_shard_power_begin(wbx_shard* s);
int wbx_shard_power_update(wbx_shard* s, int first);
int wbx_shard_power_step_a(wbx_shard* s);
int wbx_shard_power_step_t(wbx_shard* s);
/* tau = 1 / (lambda * step_safety) (1 for a zero operator) and the iteration count */
int wbx_shard_power_result(wbx_shard* s, double step_safety, double* tau, uint32_t* iters);
/* estimate_step by Lanczos (the fp32 hot path's estimator, solver.cu), device-resident; its
 * cross-rank vectors are fp32 and reuse the FISTA buffers (P^-1/2 w in y_pad, t' in res_pad):
 * lz_begin -> [all-gather sums, y] -> lz_update(0) -> repeat { lz_step_a -> [all-gather res,
 * sums] -> lz_update(1) -> lz_step_t -> [all-gather sums, y] -> lz_update(2) } -> lz_result.
 * first / every / gap: the convergence-check schedule (60 / 4 / 4 in the solver);
 * lz_done synchronises and tells the host the estimate has finished. */
int wbx_shard_lz_begin(wbx_shard* s);
int wbx_shard_lz_update(wbx_shard* s, int phase, int first, int every, int gap);
int wbx_shard_lz_step_a(wbx_shard* s);
int wbx_shard_lz_step_t(wbx_shard* s);
int wbx_shard_lz_done(wbx_shard* s, int* done);
int wbx_shard_lz_result(wbx_shard* s, double step_safety, double* tau, uint32_t* iters, uint32_t* steps);

/* ---------------------------------------------------------------- the whole sharded deblur (C4)
 * One image row-sharded over `world` ranks with the host loop, the exchange and a CUDA graph of
 * the FISTA iterations inside the library: after the first call a solve is one host call
 * (estimate_step adds one graph launch per 4 Lanczos steps from the first convergence check on).
 * The exchange is NCCL over NVLink (libnccl.so.2 resolved at run time: the one already loaded,
 * e.g. torch's, else the system's): rank 0 calls wbx_comm_get_unique_id, the caller broadcasts
 * the 128 bytes (e.g. over torch.distributed), every rank calls wbx_comm_create, then
 * wbx_sharded_create with ranks = {rank}, nranks = 1. Without a communicator all `world` ranks
 * live in this process on ctx's device and share the padded buffers (ranks = 0..world-1): the
 * partition code runs exactly as on `world` GPUs (emulation; world = 1 is the one-GPU engine).
 * Rows are summed in element order by one lane wherever they live: the restored image is
 * BITWISE the same for every world size (given tau). fp32, fixed iteration count (cfg). */
typedef struct wbx_comm wbx_comm;
int wbx_comm_get_unique_id(uint8_t* id128);
int wbx_comm_create(wbx_ctx* ctx, uint32_t world, uint32_t rank, const uint8_t* id128, wbx_comm** out);
int wbx_comm_destroy(wbx_comm* c);
typedef struct wbx_sharded wbx_sharded;
int wbx_sharded_create(wbx_ctx* ctx, uint64_t n, const uint64_t* row_offsets, const uint32_t* col_indices,
                       const double* values, wbx_basis* basis, const double* p, const double* w, double lambda,
                       const wbx_solver_cfg* cfg, uint32_t world, const uint32_t* ranks, uint32_t nranks,
                       wbx_comm* comm, wbx_sharded** out);
int wbx_sharded_destroy(wbx_sharded* s);
/* estimate_step (solver.cpp:69-99) by the sharded Lanczos estimate (WBX_TAU=power: the
 * literal power iteration); iters: the reference's iteration count; steps: product pairs */
int wbx_sharded_estimate_step(wbx_sharded* s, double step_safety, double* tau, uint32_t* iters, uint32_t* steps);
/* u0 (full image, every rank) -> analyze -> [estimate_step unless cfg.tau > 0] -> FISTA ->
 * assemble x (NCCL all-reduce of the disjoint pieces) -> synthesize (-> clamp); device
 * pointers, async on ctx's stream */
int wbx_sharded_deblur_dev(wbx_sharded* s, const double* u0_dev, double* u_dev, int clamp);
/* tau of the last deblur, its reference iteration count and product pairs, device ms of
 * (analyze + tau) and of (iterations + synthesis), kernel launches */
int wbx_sharded_stats(const wbx_sharded* s, double* tau, uint32_t* tau_iters, uint32_t* tau_steps, float* tau_ms,
                      float* iters_ms, uint64_t* launches);

/* launches of the last deblur, and the solver kernel's device time (ms) */
int wbx_solver_last_stats(const wbx_solver* s, uint64_t* launches, float* solve_ms);
// Device time of the last solve split into the step-size estimate (estimate_step, 0 when tau
// was given) and the iteration kernel(s), from CUDA events on the context stream.
int wbx_solver_phase_ms(const wbx_solver* s, float* tau_ms, float* iters_ms);
/* the step of the last solve: tau, the reference's power-iteration count for it
 * (solver.cpp:81-96) and the operator product pairs spent (Lanczos steps on the fp32 hot
 * path, power iterations otherwise; synchronises the context's stream) */
int wbx_solver_tau_stats(const wbx_solver* s, double* tau, uint32_t* ref_iters, uint32_t* product_pairs);
/* The kernels this solver runs, "<step-estimate kernel> <iteration kernel>" (NUL-terminated,
 * truncated to len): which engine the configuration and the operator selected. */
int wbx_solver_kernels(const wbx_solver* s, char* buf, uint64_t len);

#ifdef __cplusplus
}
#endif
#endif
