/*
 * mandel_dp.h -- C ABI of the Dynamic Parallelism comparison library (libmandel_dp.so).
 *
 * The paper's baseline subdivision implementation (SURVEY.md
 * §8(f) NEXT-3): the Mariani-Silver subdivision of the Mandelbrot set with
 * CUDA Dynamic Parallelism, "one kernel per node of the subdivision tree", in the
 * SBR arrangement (one block per region):
 *   - the host launches one grid of g x g blocks, one block per level-0 region;
 *   - a block computes its region's 4d-4 border dwells (written to the image), reduces
 *     (min, max) over its warps; uniform -> the block fills the region (terminal work T);
 *     else if d/r >= B -> one thread launches a CHILD GRID of r x r blocks on the
 *     region's sub-regions (device-side launch, CDP2 fire-and-forget stream); else the
 *     block computes the (d-2)^2 interior pixels itself (leaf work L).
 * The image is identical to mandel_ask's for the same (region, n, maxdwell, g, r, B): the
 * same dwell core (R2-R4) and the same decisions (R5-R7) per region; only the
 * mechanism that schedules the next level differs (recursive launches vs ASK's serial
 * level kernels over offset lists).
 *
 * Memory and ownership: d_out is a caller-owned DEVICE int32 buffer, row-major, row i at
 * d_out + i*out_pitch (out_pitch >= n); every pixel is written.  The library allocates no
 * memory itself; the CUDA device runtime keeps one pending-launch record per outstanding
 * child grid, and mandel_dp raises cudaLimitDevRuntimePendingLaunchCount (a device-wide
 * limit) to mandel_dp_pending_launches(n, g, r, B) before launching if it is lower.
 * Asynchronous on `stream` (cudaStream_t; NULL = legacy default stream): the stream's
 * work completes when every descendant grid has completed.
 *
 * Errors: MANDEL_OK, MANDEL_EINVAL (same checks as mandel_ask: n, g, r, B powers of two,
 * r >= 2, B >= 2, g*B <= n, n <= 65536, maxdwell >= 1, finite region with re_min < re_max,
 * im_min < im_max, out_pitch >= n, d_out non-null; nothing launched), MANDEL_ECUDA (a
 * runtime call or launch failed; mandel_dp_last_cuda_error() says which).  Launch failures
 * INSIDE the tree (e.g. the pending-launch limit exceeded) are reported by the next
 * synchronising CUDA call on the stream.  Codes as in mandel.h.
 */
#ifndef MANDEL_DP_H
#define MANDEL_DP_H

#include <stddef.h>
#include <stdint.h>

#include "mandel.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Upper bound of the child grids one call can have pending at once: the number of
 * subdividing nodes of the full tree, sum_{l < L-1} g^2 r^(2l) (every region may subdivide).
 * 0 for invalid parameters. */
int64_t mandel_dp_pending_launches(int64_t n, int32_t g, int32_t r, int32_t B);

/* Render the n x n dwell image of `reg` with recursive Dynamic Parallelism (see above). */
int mandel_dp(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B,
              int32_t *d_out, int64_t out_pitch, void *stream);

/* Text of the last MANDEL_ECUDA failure on this thread. */
const char *mandel_dp_last_cuda_error(void);

#ifdef __cplusplus
}
#endif

#endif /* MANDEL_DP_H */
