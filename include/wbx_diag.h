/* include/wbx_diag.h — diagnostics of libwbx (not part of the drop-in boundary). */
#ifndef WBX_DIAG_H
#define WBX_DIAG_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* Average device time (microseconds) of one grid-wide barrier of the persistent solver
 * kernels, measured over `iters` back-to-back barriers with blocks_per_sm resident CTAs
 * per SM (256 threads each). */
int wbx_diag_barrier_us(int device, int iters, int blocks_per_sm, double* us);
/* Streaming read bandwidth (GB/s) of a `bytes`-sized buffer read `reps` times by a
 * persistent grid: mode 0 = per-warp 1-D bulk copies (TMA) of `chunk` bytes into shared
 * memory with `inflight` copies in flight; mode 1 = 16-byte LDG per lane (8 in flight). */
int wbx_diag_stream_gbs(int device, int mode, uint64_t bytes, int reps, int chunk, int inflight,
                        int blocks_per_sm, double* gbs);
/* Cycle accounting of the last solves in a diagnostics build (make prof, WBX_PROFILE=3):
 * fills out[8] with the summed per-warp cycles of the window engine [A fill, A slice loop,
 * A barrier, T fill, T slice loop, T barrier, 0, 0] and resets the counters. */
int wbx_diag_slice_profile(double* out);
/* The fp32 SELL kernel of wbx_spmv_compact_dev selected explicitly (tests compare the
 * variants; WBX_SPMV selects the default once per process): mode 0 reg, 1 tma1, 2 tma2,
 * 3 tma3, 4 half, 5 quarter (segmented layout, one fma order), 6 row2, 7 row (default),
 * 8 row8 (row-per-lane layout, element order). Device pointers, compacted spaces, async. */
struct wbx_ctx;
struct wbx_op;
/* L2 prefetch distance (bytes ahead in the operator stream) of the row kernel; -1 restores
 * the default (WBX_SPMV_PF, else 0 = no prefetch: measured slower on B200). */
int wbx_diag_set_spmv_pf(long long bytes);
int wbx_diag_spmv_compact_mode(struct wbx_ctx* ctx, const struct wbx_op* op, int transpose, int mode,
                               const float* x_dev, float* y_dev);
/* Per-CTA features of a solver's window layout (side 0: Theta rows, 1: Theta^T rows):
 * out[G][6] = {rows, sum 1/m, sum nq/m, sum (q-1)/m, nonzeros, window entries}. */
/* Host execution of the stencil engine's plan (grid G) for an operator given by its kept
 * generator groups: y = Theta x (phase 0) / Theta^T x (phase 1), full-length fp64 vectors. */
int wbx_diag_stencil_apply_host(uint32_t ndim, const uint64_t* dims, uint32_t J, uint64_t n_gens,
                                const uint32_t* blocks, const uint32_t* gen_index, const uint64_t* counts,
                                const double* values, int phase, uint32_t G, const double* x, double* y);
/* Block-Fourier step estimate (csrc/circ_tau.cu): does it apply to `op` on the layout
 * (ndim, dims, J)? info[5] = {applies, row orbits, column orbits, g0, g1}; `why` gets the reason
 * when it does not (host analysis, cached on the operator). */
int wbx_diag_circ_info(const struct wbx_op* op, uint32_t ndim, const uint64_t* dims, uint32_t J, uint32_t* info,
                       char* why, uint64_t why_len);
struct wbx_solver;
int wbx_diag_win_features(const struct wbx_solver* s, int side, double* out, int* G);
#ifdef __cplusplus
}
#endif
#endif
