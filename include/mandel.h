/*
 * mandel.h -- C ABI of the B200 ASK Mandelbrot library (libmandel_b200.so).
 *
 * The operations are the paper's (P:NNN = /root/reference/PAPER.md line NNN):
 *   mandel_exhaustive   the exhaustive approach Ex: one flat kernel, one thread per pixel
 *                       (P:111-117 eq:exhaustive-general; "Ex: Exhaustive approach in
 *                       one flat kernel execution").
 *   mandel_ask          Adaptive Serial Kernels (Sec. 5) applied to the
 *                       Mariani-Silver subdivision of the Mandelbrot set:
 *                       initial g x g regions, border dwell per region, fill if the border is
 *                       uniform, else split r x r while the child side stays >= B, else
 *                       per-pixel dwell (leaf).  "Generating the Mandelbrot set in the complex
 *                       plane [region] using a dwell of d ... problem size n x n".
 *   mandel_ask_tiles    mandel_ask restricted to a subset of the level-0 regions (the
 *                       multi-GPU partition: each rank runs its own tiles).
 *
 * Arithmetic (R2-R4): dwell = first i >= 1 with |z_i|^2 > 4 (z_0 = 0), else
 * maxdwell; IEEE binary32, round-to-nearest, no FMA contraction, no FTZ, operation order
 * x2=x*x, y2=y*y, xy=x*y, x=(x2-y2)+cr, y=(xy+xy)+ci.  Pixel (row i, column j) samples
 * its centre c = cr + i ci with cr = (float)re_min + ((float)j+0.5f)*dx and
 * ci = (float)im_min + ((float)i+0.5f)*dy, dx = (float)((re_max-re_min)/n), dy likewise
 * (each a single RN float operation); row i = 0 is the im_min side.
 *
 * Memory and ownership:
 *   - d_out: caller-owned DEVICE buffer of int32, row-major, row i at d_out + i*out_pitch
 *     (out_pitch >= n elements).  mandel_exhaustive and mandel_ask write every pixel;
 *     mandel_ask_tiles writes only the pixels of its tiles.  The vectorised fill needs
 *     d_out 16-byte aligned and out_pitch % 4 == 0; other layouts fall back to 4-byte stores.
 *   - d_ws: caller-owned DEVICE workspace of >= mandel_ask_workspace_bytes(...) bytes
 *     (device parameter block, offset lists, fill/leaf lists, counters).  One in-flight call
 *     per workspace.
 *   - The library never allocates device memory.  It caches one captured CUDA graph per
 *     launch shape -- key (device, n, out_pitch, g, r, B, scheme, flags, d_out, d_ws,
 *     ws_bytes, number of tiles, whether a tile list is given) -- and frees them in
 *     mandel_shutdown().  The region, maxdwell and the tile ids are NOT part of the key: every
 *     call first writes them into a parameter block inside d_ws with one stream-ordered
 *     host->device copy (staged from pageable memory, so the caller's arrays are free on
 *     return), and the graph's kernels read them there.  One graph therefore serves every
 *     view, maxdwell and tile list of a launch shape (the ASK state is kept
 *     device-resident; the paper's host loop reads `count` back after every level).
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream),
 *     except mandel_ask_last_stats, which synchronises it.
 *
 * Errors: every function returns MANDEL_OK or an error code and never throws.
 *   MANDEL_EINVAL      invalid argument (checked synchronously, nothing launched):
 *                      n, g, r, B powers of two; r >= 2; B >= 2; g*B <= n; n <= 65536;
 *                      1 <= maxdwell; re_min < re_max, im_min < im_max (finite);
 *                      out_pitch >= n; non-null pointers; tile ids in [0, g*g), unique.
 *   MANDEL_EWORKSPACE  ws_bytes < mandel_ask_workspace_bytes(...).
 *   MANDEL_ECUDA       a CUDA runtime call or launch failed (see mandel_last_cuda_error()).
 */
#ifndef MANDEL_B200_H
#define MANDEL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Complex-plane window, SPEC.md S:173-176 Viewport.  */
typedef struct {
    double re_min, re_max, im_min, im_max;
} mandel_region;

/* Per-level statistics (SPEC.md S:274-277 LevelStats, extended with pixel counts). */
typedef struct {
    int32_t level;        /* 0 = the initial g x g split                                    */
    int32_t side;         /* region side d at this level: n/(g r^level)                     */
    int64_t regions_in;   /* regions examined (= |G_level|)                          */
    int64_t filled;       /* uniform border -> filled (terminal work T)              */
    int64_t subdivided;   /* non-uniform, d/r >= B -> r*r children              */
    int64_t leaves;       /* non-uniform, d/r <  B -> per-pixel dwell (L)        */
    int64_t border_px;    /* border pixels whose dwell this level computed                  */
    int64_t border_iters; /* iterations counted for them (= sum of their dwells)            */
    int64_t leaf_px;      /* leaf interior pixels computed at this level                    */
    int64_t leaf_iters;   /* sum of their dwells                                           */
} mandel_level_stats;

enum {
    MANDEL_OK = 0,
    MANDEL_EINVAL = 1,
    MANDEL_EWORKSPACE = 2,
    MANDEL_ECUDA = 3
};

/* Scheme of the subdivision kernels.  All produce bit-identical images.
 *   MANDEL_SCHEME_SBR   the paper's ASK-SBR, "single block per region" (P:296-302,
 *                       P:366-377): per level one CUDA kernel in which one block per region
 *                       computes the region's whole border (query Q, split across its
 *                       warps, reduced with warp reductions), appends to the next-level
 *                       offset list or the leaf list (PS), and fills the region itself when
 *                       the border is uniform (Delta[T]); leaves: one block each (Delta[L]).
 *                       1 + L + 1 kernels per call.
 *   MANDEL_SCHEME_B200  B200 re-design: border dwells are written to the
 *                       image and reused -- a child only computes the new internal division
 *                       lines of its parent -- by a flat, load-balanced kernel over all new
 *                       border pixels of the level; a warp per region then decides
 *                       uniformity from the image with warp reductions; leaf interiors run
 *                       as one flat pixel-parallel kernel.  1 + 3L + 1 kernels.
 *   MANDEL_SCHEME_MBR   the paper's ASK-MBR, "multiple blocks per region": Q and
 *                       PS as in SBR (block per region), terminal work T and leaf work L as
 *                       flat multi-block kernels over all regions of the level (nabla[T],
 *                       nabla[L]), one thread per pixel.  1 + 2L + 1 kernels.
 */
enum {
    MANDEL_SCHEME_SBR = 0,
    MANDEL_SCHEME_B200 = 1,
    MANDEL_SCHEME_MBR = 2
};

/* flags */
#define MANDEL_FLAG_STATS 1u  /* also accumulate border/leaf pixel + iteration counters   */
#define MANDEL_FLAG_TIMING 2u /* record a CUDA event after every kernel of the call (graph
                                 event-record nodes) for mandel_ask_kernel_times()          */
#define MANDEL_FLAG_TILE_COST 4u /* accumulate executed iterations per level-0 tile for
                                    mandel_ask_tile_costs() (per-pixel atomics: preview use) */
#define MANDEL_FLAG_FLAT 8u      /* B200 scheme: plain one-thread-per-pixel border and leaf
                                    kernels instead of the lane-refill ones (A/B baseline;
                                    same image)                                            */
/* Like MANDEL_FLAG_TILE_COST, but estimated, and a time proxy rather than an iteration count:
 * only the pixels on the lattice (x + y) mod 64 == 0 are counted, each as 64 * (dwell + 64) --
 * its iterations plus 64 for the engine's per-pixel work (B200 scheme, refill kernels;
 * elsewhere, or together with MANDEL_FLAG_STATS / MANDEL_FLAG_TILE_COST, the call counts
 * exact iterations).  At 1/64 of the counting work: the multi-GPU deal's per-step feedback
 * (DESIGN.md §9).                                                                            */
#define MANDEL_FLAG_TILE_COST_SAMPLED 32u
#define MANDEL_FLAG_SERIAL 16u   /* run every fill on the main stream after its level instead
                                    of as a concurrent graph branch (A/B; same image)       */
/* Groups: the call's level-0 tiles are dealt round-robin (in the given order) to G independent
 * ASK chains, each level-synchronous, captured as parallel graph branches, so one chain's
 * level tails overlap another's work.  G in {1..8}, encoded in flag bits
 * 8-11 as G-1; 0 there means 1 group.  Same image for every G.                           */
#define MANDEL_FLAG_GROUPS(G) ((((uint32_t)(G)-1u) & 15u) << 8)
#define MANDEL_FLAG_GROUPS_MASK (15u << 8)
#define MANDEL_FLAG_GROUPS_OF(f) ((int)(((f) >> 8) & 15u) + 1)
/* Like MANDEL_FLAG_TIMING, but events only around the leaf kernel (the dominant one): the
 * event nodes of MANDEL_FLAG_TIMING sit between every pair of kernels and so cut the
 * programmatic-dependent-launch edges of the level chain.                 */
#define MANDEL_FLAG_TIMING_LEAF 128u

/* Kernel kinds reported by mandel_ask_kernel_times (value = kind * 100 + level). */
enum {
    MANDEL_KIND_INIT = 0,          /* level-0 offset list + counters                          */
    MANDEL_KIND_B200_BORDER = 1,   /* new border pixels of a level (dwell)                    */
    MANDEL_KIND_B200_CLASSIFY = 2, /* warp-per-region uniformity test + list appends          */
    MANDEL_KIND_FILL = 3,          /* fill of the level's uniform regions                     */
    MANDEL_KIND_B200_LEAF = 4,     /* leaf interiors, flat                                    */
    MANDEL_KIND_SBR_LEVEL = 5,     /* paper SBR/MBR: block-per-region border + decision       */
    MANDEL_KIND_SBR_LEAF = 6,      /* paper SBR: block-per-leaf interior                      */
    MANDEL_KIND_MBR_LEAF = 7       /* paper MBR: leaf interiors, flat multi-block             */
};

/* Bytes of workspace mandel_ask / mandel_ask_tiles need for these parameters (worst case
 * over all images: every region at every level may subdivide).  0 if invalid. */
size_t mandel_ask_workspace_bytes(int64_t n, int32_t g, int32_t r, int32_t B);

/* Number of subdivision levels ASK runs: 1 + floor(log_r((n/g)/B)).  0 if invalid. */
int32_t mandel_ask_levels(int64_t n, int32_t g, int32_t r, int32_t B);

/* Exhaustive dwell image Ex. */
int mandel_exhaustive(mandel_region reg, int64_t n, int32_t maxdwell, int32_t *d_out,
                      int64_t out_pitch, void *stream);

/* The same exhaustive image from a tuned flat kernel: one thread per pixel as well, but the
 * escape test runs every 32 iterations instead of 8 (less per-chunk bookkeeping; the exact
 * first-escape index is still recovered by replaying the last chunk) and 32 x 8 blocks.  It is
 * the second, fairer speedup denominator SURVEY.md §8(d) asks for beside the plain kernel.
 * Same arguments, same image. */
int mandel_exhaustive_tuned(mandel_region reg, int64_t n, int32_t maxdwell, int32_t *d_out,
                            int64_t out_pitch, void *stream);

/* Full ASK image over all g*g level-0 regions. */
int mandel_ask(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B,
               int32_t *d_out, int64_t out_pitch, void *d_ws, size_t ws_bytes, void *stream);

/* ASK over the level-0 regions h_tile_ids[0..n_tiles) (HOST array; canonical id
 * k = gy*g + gx), with an explicit scheme and flags.  n_tiles == 0 with h_tile_ids == NULL
 * means all g*g tiles in canonical order. */
int mandel_ask_tiles(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r,
                     int32_t B, const int32_t *h_tile_ids, int32_t n_tiles, int32_t scheme,
                     uint32_t flags, int32_t *d_out, int64_t out_pitch, void *d_ws,
                     size_t ws_bytes, void *stream);

/* mandel_ask_tiles with the tile list in DEVICE memory: d_tile_ids (>= g*g int32 entries) and
 * its length *d_n_tiles (int32) are read when the call executes on `stream`, not when it is
 * enqueued -- the captured graph copies them into the workspace's parameter block itself -- so a
 * preceding kernel on the stream (mandel_deal_lpt) can choose the tiles and no host round trip is
 * needed between the multi-GPU deal and the rank's ASK.  The graph is keyed on the two pointers,
 * not on the count.  Ids must be unique and in [0, g*g) (not checked on the device).
 * MANDEL_FLAG_GROUPS must be 1; g*g <= 4096. */
int mandel_ask_dtiles(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r,
                      int32_t B, const int32_t *d_tile_ids, const int32_t *d_n_tiles, int32_t scheme,
                      uint32_t flags, int32_t *d_out, int64_t out_pitch, void *d_ws, size_t ws_bytes,
                      void *stream);

/* The multi-GPU partition (north_star "initial g x g regions dealt across
 * ranks"; P:366 the level-0 grid |G_0|), on the device: Graham's longest-processing-time list
 * schedule of n_tiles level-0 tiles over `world` ranks on the per-tile costs d_costs (u64,
 * canonical tile order): tiles in descending cost (ties: lower id), each to the least-loaded rank
 * (ties: lower rank).  Writes rank `rank`'s tiles, in that descending order, to d_tile_ids and
 * their number to *d_n_tiles (device memory), asynchronously on `stream`.  Deterministic: every
 * rank computing it on the same costs gets a consistent partition.  n_tiles <= 4096,
 * world <= 64. */
int mandel_deal_lpt(const uint64_t *d_costs, int32_t n_tiles, int32_t world, int32_t rank,
                    int32_t *d_tile_ids, int32_t *d_n_tiles, void *stream);

/* Byte offset, inside a workspace of these parameters, of the per-tile executed-iteration
 * counters (u64[g*g], canonical order) that MANDEL_FLAG_TILE_COST fills; lets the caller reduce
 * them across ranks in place (e.g. NCCL all-reduce) and feed mandel_deal_lpt.  0 if invalid. */
size_t mandel_ask_tile_costs_offset(int64_t n, int32_t g, int32_t r, int32_t B);

/* End-to-end variant over HOST memory: runs mandel_ask_tiles into the device buffer d_out
 * and copies the n x n image (rows of n elements) into h_out (host; pinned for full
 * bandwidth), then synchronises `stream`.  For tile runs only the tiles' pixels are
 * meaningful.  h_out is written with row pitch n.  For the whole image (h_tile_ids NULL) the
 * call is pipelined: min(g, 8) bands of level-0 tile rows run as separate tile calls and the
 * copy of each band overlaps the computation of the next (same image: level-0 regions are
 * independent).  One call at a time per device. */
int mandel_ask_to_host(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r,
                       int32_t B, const int32_t *h_tile_ids, int32_t n_tiles, int32_t scheme,
                       int32_t *d_out, int64_t out_pitch, void *d_ws, size_t ws_bytes,
                       int32_t *h_out, void *stream);

/* mandel_ask_to_host with a 16-bit host image: the same call and pipeline, but every finished
 * band (or tile) is first narrowed on the device into d_stage -- caller-owned DEVICE buffer of
 * n*n uint16, row pitch n -- and the copy reads d_stage, so the host receives n*n uint16
 * (h_out, row pitch n; ideally pinned) and PCIe carries half the bytes.  Dwells lie in
 * [1, maxdwell], so the narrowing is exact; maxdwell > 65535 or a NULL d_stage is
 * MANDEL_EINVAL.  d_out still receives the int32 image. */
int mandel_ask_to_host_u16(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r,
                           int32_t B, const int32_t *h_tile_ids, int32_t n_tiles, int32_t scheme,
                           int32_t *d_out, int64_t out_pitch, void *d_ws, size_t ws_bytes,
                           uint16_t *d_stage, uint16_t *h_out, void *stream);

/* Per-level statistics of the last call that used d_ws (synchronises `stream`).
 * Writes min(levels, max_levels) entries; returns the number of levels (>= 0) or -code. */
int mandel_ask_last_stats(const void *d_ws, mandel_level_stats *h_out, int32_t max_levels,
                          void *stream);

/* Device time of every kernel of the most recent mandel_ask_tiles call made with
 * MANDEL_FLAG_TIMING (waits for it to finish).  Writes up to max_kernels entries of ms[]
 * (milliseconds, may be NULL) and kind_level[] (may be NULL); returns the kernel count or
 * -code. */
int mandel_ask_kernel_times(float *ms, int32_t *kind_level, int32_t max_kernels);

/* Executed iterations per level-0 tile (canonical id order, g*g entries, u64) of the last
 * call on d_ws made with MANDEL_FLAG_TILE_COST (synchronises `stream`).  Writes up to
 * max_tiles entries; returns g*g or -code.  Used to rank tiles for the multi-GPU deal. */
int mandel_ask_tile_costs(const void *d_ws, uint64_t *h_costs, int32_t max_tiles, void *stream);

/* Number of kernel launches one mandel_ask_tiles call issues for these parameters. */
int32_t mandel_ask_kernel_count(int64_t n, int32_t g, int32_t r, int32_t B, int32_t scheme);

/* Number of CUDA graphs captured and instantiated by this process so far (one per new launch
 * shape, see "Memory and ownership"); lets a caller check that repeated calls with other
 * regions, maxdwell values or tile lists reuse one graph. */
long long mandel_ask_graph_captures(void);

/* Measurement helper (not a step of the method): the FP32 issue rate of the dwell step on
 * this device -- the paper's machine model charges q processors x c lanes, and
 * bench.py divides the dwell kernels' algorithmic FP32 ops by this measured rate.  Runs the
 * 7-op step of the dwell core on 2 independent non-escaping orbits per thread, 8 x 256
 * threads per SM, `steps` x 8 steps each (4 runs, the first a warm-up), synchronously on
 * `stream`; writes the best rate in T FP32 ops/s (one FADD or FMUL = 1 op) to *tops. */
int mandel_fp32_peak_probe(int32_t steps, double *tops, void *stream);

const char *mandel_strerror(int code);
const char *mandel_last_cuda_error(void);
void mandel_shutdown(void); /* frees cached graphs/events/streams; owns no device buffers */

#ifdef __cplusplus
}
#endif
#endif /* MANDEL_B200_H */
