/*
 * mandel3d.h -- C ABI of libmandel3d.so: ASK on k = 3 orthotopes (NEXT-4; the paper's
 * Sec. 6.2 "Subdivisions at Higher Dimensions"), hand-written sm_100a kernels.
 *
 * The paper sketches ASK for k >= 3 (g^k initial regions, r^k sub-orthotopes per subdividing
 * region; OLT size |T_i^k| = |G_i| prod_j r_j; one SFC scalar per OLT
 * entry instead of k coordinates) without a workload.  DESIGN.md §12, readings
 * R15-R17, fix the one computed here:
 *   - the volume is the (c_re, c_im, w) slice of the quadratic family's parameter space:
 *     z_{i+1} = z_i^2 + c from z_0 = w + 0i; dwell = first i >= 1 with |z_i|^2 > 4, else
 *     maxdwell, FP32 round-to-nearest without FMA in the operation order of include/mandel.h
 *     (bit-identical to the oracle);
 *   - voxel (x, y, z) samples its centre on each axis exactly like the 2-D pixel mapping;
 *   - a region's border is its surface (voxels with a coordinate on the cube's boundary);
 *     uniform surface -> fill the cube; else d/r >= B -> r^3 sub-cubes; else every voxel.
 *
 * Layout: the n x n x n int32 volume is dense, voxel (x, y, z) at out[(z * n + y) * n + x],
 * i.e. the canonical-order SFC Omega(p) = n^2 p_z + n p_y + p_x of the voxel;
 * the OLT stores that scalar of each region's corner voxel (u32: n <= 1024).
 * Ownership: the caller owns d_out (device, 4 n^3 bytes) and d_ws (device, 256-byte
 * aligned, mandel3d_ask_workspace_bytes()); calls are asynchronous on `stream` (a
 * cudaStream_t, NULL = legacy default stream), one in flight per workspace.
 * Errors: 0 ok; 1 invalid argument (n, g, r, B powers of two, r >= 2, B >= 2, g*B <= n,
 * n <= 1024, 1 <= maxdwell, min < max on every axis, non-null pointers) -- checked before any
 * CUDA call; 2 workspace too small; 3 CUDA error (mandel3d_last_cuda_error()).
 */
#ifndef MANDEL3D_H
#define MANDEL3D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double re_min, re_max, im_min, im_max, w_min, w_max;
} mandel3d_region;

typedef struct {
    int32_t level, side;
    int64_t regions_in;   /* regions examined at this level                                  */
    int64_t filled;       /* uniform surface -> filled                                       */
    int64_t subdivided;   /* -> r^3 regions at level + 1                                     */
    int64_t leaves;       /* -> every voxel computed                                         */
    int64_t border_px;    /* surface voxels computed at this level (MANDEL3D_FLAG_STATS)     */
    int64_t border_iters; /* sum of their dwells (MANDEL3D_FLAG_STATS)                       */
    int64_t leaf_px;      /* leaf interior voxels computed (MANDEL3D_FLAG_STATS)             */
    int64_t leaf_iters;   /* sum of their dwells (MANDEL3D_FLAG_STATS)                       */
} mandel3d_level_stats;

#define MANDEL3D_FLAG_STATS 1u /* also accumulate the voxel / iteration counters            */
#define MANDEL3D_FLAG_FLAT 2u  /* plain thread-per-voxel surface and leaf kernels instead of
                                  the lane-refill ones (A/B; same volume)                    */

/* Workspace bytes for these parameters (0: invalid).  Worst case: every region subdivides. */
size_t mandel3d_ask_workspace_bytes(int64_t n, int32_t g, int32_t r, int32_t B);

/* Subdivision levels: 1 + floor(log_r((n/g)/B)) (0: invalid). */
int32_t mandel3d_ask_levels(int64_t n, int32_t g, int32_t r, int32_t B);

/* Exhaustive volume: one thread per voxel (the speedup denominator). */
int mandel3d_exhaustive(mandel3d_region reg, int64_t n, int32_t maxdwell, int32_t *d_out, void *stream);

/* 3-D ASK volume over all g^3 level-0 cubes: per level a surface kernel (lane-refill engine of
 * DESIGN.md §4.6 over voxels, or MANDEL3D_FLAG_FLAT thread-per-voxel; level 0: every
 * surface voxel of every region; deeper levels: only the division-plane voxels of each
 * subdivided parent, the rest of the children's surfaces being the parent's, already in the
 * volume), a block-per-region classification (min/max reduction;
 * fill list / r^3 OLT slots by one atomicAdd / leaf list), a flat 128-bit fill of the
 * uniform cubes, and a flat kernel over the leaves' interior voxels at the end; region
 * counts stay in device memory (no host round trip). */
int mandel3d_ask(mandel3d_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B,
                 uint32_t flags, int32_t *d_out, void *d_ws, size_t ws_bytes, void *stream);

/* Per-level statistics of the last mandel3d_ask on d_ws (synchronises `stream`); returns the
 * level count or -code. */
int mandel3d_ask_last_stats(const void *d_ws, mandel3d_level_stats *h_out, int32_t max_levels, void *stream);

const char *mandel3d_last_cuda_error(void);
void mandel3d_shutdown(void); /* frees the per-device fill stream and events; owns no buffers */

#ifdef __cplusplus
}
#endif
#endif /* MANDEL3D_H */
