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
#ifdef __cplusplus
}
#endif
#endif
