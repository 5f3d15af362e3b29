// ask_kernels.cuh -- sm_100a kernels of the exhaustive baseline and the ASK level loop.
//
// P:NNN = /root/reference/PAPER.md line NNN.  Data layout in HBM:
//   image   int32 row-major, pixel (row y, column x) at out[y*pitch + x]
//   OLT     u32 packed region origin (x | y << 16), two ping-pong buffers
//   fill    uint2 {packed origin, fill value}, one segment per level
//   leaf    u32 packed origin of the last level's non-uniform regions
//   header  counters: subdivided / filled per level, leaves, optional iteration stats
#pragma once
#include <limits.h>
#include <stddef.h>
#include <stdint.h>

#include "dwell.cuh"
#include "refill.cuh"

namespace mandel {

constexpr int MAXL = 32;
constexpr int MAXG = 8; // independent ASK chains (groups) per call
constexpr uint32_t WS_MAGIC = 0x4d41534bu; // "MASK"
constexpr int DWELL_K = 8;                 // iterations per escape test (dwell.cuh)
// Lane-refill knobs (refill.cuh), tuned on B200 at C3/C5 (profiles/r01_tune_refill*.txt):
// K iterations per escape test, T parked lanes that trigger a warp refill, CH indices a warp
// grabs per cursor atomic; separately for the border (short, level-synchronous launches:
// smaller grabs balance better) and leaf kernels.
#ifndef MANDEL_RFB_K
#define MANDEL_RFB_K 32
#endif
#ifndef MANDEL_RFB_T
#define MANDEL_RFB_T 8
#endif
#ifndef MANDEL_RFB_CH // border grab cap (128: C4 -0.9%, C5 -0.3%, C3 -0.25% against 64;
#define MANDEL_RFB_CH 128 // profiles/r02_ab_border_ch_t.jsonl)
#endif
#ifndef MANDEL_RFB_CH_DEV // ... and for device-tile-list calls (one rank's share of the N > 1 step),
#define MANDEL_RFB_CH_DEV 64 // where 128 unbalanced the 8-way C4 deal (6.85x vs 7.07x emulated)
#endif
#ifndef MANDEL_RFL_K
#define MANDEL_RFL_K 32
#endif
#ifndef MANDEL_RFL_T
#define MANDEL_RFL_T 8
#endif
#ifndef MANDEL_RFL_CH
#define MANDEL_RFL_CH 128
#endif
#ifndef MANDEL_RF_MINB
#define MANDEL_RF_MINB 4
#endif
// Packed engine (refill_loop2, two pixels per lane on FFMA2/FADD2): on/off per kernel, T out
// of 64 slots, resident blocks per SM.  Measured on B200 (profiles/r01_tune_refill_v3.txt):
// packed for the leaves (fewer bookkeeping instructions per pixel), scalar for the border
// levels (a level's tail is one long pixel's latency, and a scalar warp steps a pixel twice
// as fast as a packed one when the SM has drained).
#ifndef MANDEL_RFB_PACK
#define MANDEL_RFB_PACK 0
#endif
#ifndef MANDEL_RFL_PACK
#define MANDEL_RFL_PACK 1
#endif
#ifndef MANDEL_RFB2_T
#define MANDEL_RFB2_T 8
#endif
#ifndef MANDEL_RFL2_T
#define MANDEL_RFL2_T 8
#endif
#ifndef MANDEL_RF2_MINB
#define MANDEL_RF2_MINB 3
#endif
// Short-pixel prepass steps of the packed leaf engine (refill.cuh rf2_prepass; 0 = off).
#ifndef MANDEL_RFL_PRE
#define MANDEL_RFL_PRE 16
#endif
#ifndef MANDEL_RFB_PRE
#define MANDEL_RFB_PRE 16 // (packed border engine only)
#endif
#ifndef MANDEL_RF_TPB
#define MANDEL_RF_TPB 256
#endif
#ifndef MANDEL_RFB_SPRE // scalar border engine: short-pixel prepass steps (0: off)
#define MANDEL_RFB_SPRE 0
#endif
#ifndef MANDEL_HOT_SHIFT // longest-first split: "hot" iff ring max >= maxdwell >> SHIFT
#define MANDEL_HOT_SHIFT 1
#endif
#ifndef MANDEL_PDL
#define MANDEL_PDL 1
#endif
constexpr int RF_TPB = MANDEL_RF_TPB;                    // threads per refill block
constexpr int RF_MINB = MANDEL_RF_MINB * (256 / RF_TPB); // resident blocks per SM (register cap)
constexpr int RFB_MINB = MANDEL_RFB_PACK ? MANDEL_RF2_MINB * (256 / RF_TPB) : RF_MINB;
constexpr int RFL_MINB = MANDEL_RFL_PACK ? MANDEL_RF2_MINB * (256 / RF_TPB) : RF_MINB;

struct WsHeader {
    uint32_t magic, levels, n, g, r, B, ntiles, scheme; // written by k_init
    uint32_t n_subdiv[MAXL];                           // OLT "count" per level
    uint32_t n_fill[MAXL];
    uint32_t n_leaf;
    uint32_t pad0;
    // Longest-first ordering: subdivided parents and leaves are appended to 4
    // length buckets by the share of their ring at maxdwell (bucket 3: >= 1/2, 2: >= 1/8, 1:
    // ring max >= maxdwell/2, 0: the rest); the next kernel hands out bucket 3 first.
    uint32_t n_sub_b[MAXL][4];
    uint32_t n_leaf_b[4];
    uint32_t ngroups; // header of group 0: groups of the last call
    unsigned long long border_px[MAXL], border_iters[MAXL];
    unsigned long long leaf_px, leaf_iters;
    unsigned long long cursor[MAXL + 1]; // lane-refill work cursors: border level l, leaves
};
static_assert(sizeof(WsHeader) <= 4096, "header");

__device__ __forceinline__ uint32_t pack_xy(int x, int y) { return (uint32_t)x | ((uint32_t)y << 16); }
__device__ __forceinline__ int unpack_x(uint32_t o) { return (int)(o & 0xffffu); }
__device__ __forceinline__ int unpack_y(uint32_t o) { return (int)(o >> 16); }

// Border pixel b in [0, 4d-4) of the region with origin (x0, y0) and side d: top row,
// bottom row, then the left and right columns without their corners (each pixel once).
__device__ __forceinline__ void ring_pixel(int b, int d, int x0, int y0, int &x, int &y)
{
    if (b < d) {
        x = x0 + b;
        y = y0;
    } else if (b < 2 * d) {
        x = x0 + (b - d);
        y = y0 + d - 1;
    } else if (b < 3 * d - 2) {
        x = x0;
        y = y0 + 1 + (b - 2 * d);
    } else {
        x = x0 + d - 1;
        y = y0 + 1 + (b - (3 * d - 2));
    }
}

struct ExArgs {
    PixMap map;
    int n, maxdwell;
    long long pitch;
    int *out;
};

// Per-call parameters in the workspace: the host writes them with one
// stream-ordered copy before every graph launch, so one captured graph serves any region,
// maxdwell and tile list (the OLT state stays device-resident between calls).
struct DevParams {
    PixMap map;       // pixel -> c of the call's region (dwell.cuh, R3)
    int32_t maxdwell; // >= 1
    uint32_t magic;   // PRM_MAGIC
    int32_t ntiles;   // level-0 tiles of the call (host lists: the graph is keyed on it; device
                      // lists: copied from the caller's device counter by the graph itself)
    uint32_t pad;
    // followed at byte offset PRM_TILES by the call's tile list (int32, group-dealt order)
};
constexpr size_t PRM_HOST_BYTES_DTILES = 24; // host-written part for device tile lists
constexpr uint32_t PRM_MAGIC = 0x4d505242u; // "BRPM"
constexpr size_t PRM_TILES = 256;

struct LevelArgs {
    PixMap map;              // filled from *prm at kernel entry (with_params)
    int maxdwell;            // filled from *prm at kernel entry
    const DevParams *prm;    // device parameter block of the call
    long long pitch;
    int *out;
    WsHeader *hdr;
    const uint32_t *olt_in;  // regions of this level
    uint32_t *olt_out;       // children for the next level
    uint2 *fill;             // this level's fill segment
    uint32_t *leaf;
    const int32_t *tiles;    // k_init only: the group's tile list in the parameter block (NULL: canonical)
    const int32_t *src_tiles, *src_ntiles; // k_init only: the caller's device tile list and length
                                           // (mandel_ask_dtiles, one group), copied by k_init
    int zero_costs;          // k_init only: zero the g*g tile-cost counters (one group)
    int level, d, r, B, g, ntiles, levels, scheme; // ntiles < 0: read prm->ntiles (device list)
    int subdivide;           // d / r >= B
    int log2_q4, log2_row4;  // fill: log2(d*d/4), log2(d/4)
    int fill_vec;            // SBR in-block fill: rows 16-byte aligned and d % 4 == 0
    unsigned long long *tile_cost; // MANDEL_FLAG_TILE_COST: iterations per level-0 tile
    int d0;                  // level-0 side
    int d0_log2, g_log2;     // d0 = n/g and g are powers of two: tile of (x, y) by shifts
    // Column lines, transposed (B200 scheme, leaf side u >= 8): every pixel
    // on a column x with x mod u in {0, u-1} -- the only columns any region ring uses -- is
    // also stored at colT[(2 (x / u) + (x mod u != 0)) * colT_pitch + y], so classification
    // reads ring columns as contiguous runs instead of one 32-byte image sector per pixel.
    int *colT;               // NULL: classify reads columns from the image
    int u_log2;
    long long colT_pitch;    // = n
    FastDiv fd[4];           // lane-refill index maps (host-computed divisors)
    uint32_t capP;           // parent slots of one bucket block of an OLT buffer
    uint32_t capL;           // leaf entries of one bucket block of the leaf list
    int ngroups;
    int pdl_late;            // refill kernels trigger their successor in the tail (device tile list)
};

// Length-bucket list addressing.  A list (subdivided parents of a level, or
// leaves) lives in two two-ended blocks of `cap` slots: bucket 3 from the front of block A,
// bucket 2 from its back, bucket 1 from the front of block B, bucket 0 from its back.  A
// consumer walks it in bucket order 3, 2, 1, 0 (longest work first); `slot(q)` is the slot of
// the q-th entry in that order, `put(b, e)` the slot of the e-th entry appended to bucket b.
struct BucketMap {
    uint32_t e3, e32, e321; // prefix ends of buckets 3, 3+2, 3+2+1 in consumption order
    uint32_t cap;
    __device__ __forceinline__ uint32_t slot(uint32_t q) const
    {
        if (q < e3)
            return q;
        if (q < e32)
            return cap - 1u - (q - e3);
        if (q < e321)
            return cap + (q - e32);
        return 2u * cap - 1u - (q - e321);
    }
};
__device__ __forceinline__ uint32_t bucket_put(int b, uint32_t e, uint32_t cap)
{
    return b == 3 ? e : b == 2 ? cap - 1u - e : b == 1 ? cap + e : 2u * cap - 1u - e;
}
__device__ __forceinline__ BucketMap bucket_map(const uint32_t *cnt, uint32_t cap)
{
    const volatile uint32_t *c = cnt;
    BucketMap m;
    m.e3 = c[3];
    m.e32 = m.e3 + c[2];
    m.e321 = m.e32 + c[1];
    m.cap = cap;
    return m;
}
// Parents of this level's regions (level > 0); level 0 reads the tile list in order.
__device__ __forceinline__ BucketMap sub_buckets(const LevelArgs &a)
{
    if (a.level == 0) {
        BucketMap m{0xffffffffu, 0xffffffffu, 0xffffffffu, a.capP};
        return m;
    }
    return bucket_map(a.hdr->n_sub_b[a.level - 1], a.capP);
}
__device__ __forceinline__ BucketMap leaf_buckets(const LevelArgs &a) { return bucket_map(a.hdr->n_leaf_b, a.capL); }
// The ri-th region of this level (children of the q-th parent are r^2 consecutive entries).
__device__ __forceinline__ uint32_t region_origin(const LevelArgs &a, uint32_t ri, const BucketMap &bm)
{
    if (a.level == 0)
        return a.olt_in[ri];
    const uint32_t rr = (uint32_t)(a.r * a.r), q = ri / rr;
    return a.olt_in[(size_t)bm.slot(q) * rr + (ri - q * rr)];
}
// Length bucket of a region from its ring: nmax of its `ring` pixels sit at maxdwell, hi = max.
__device__ __forceinline__ int length_bucket(const LevelArgs &a, int hi, int nmax, int ring)
{
    if (2 * nmax >= ring)
        return 3;
    if (8 * nmax >= ring)
        return 2;
    return ((long long)hi << MANDEL_HOT_SHIFT) >= a.maxdwell ? 1 : 0;
}

__device__ __forceinline__ bool on_col_line(const LevelArgs &a, int x)
{
    const int m = x & ((1 << a.u_log2) - 1);
    return m == 0 || m == (1 << a.u_log2) - 1;
}
__device__ __forceinline__ long long colT_index(const LevelArgs &a, int x, int y)
{
    const int m = x & ((1 << a.u_log2) - 1);
    return (long long)(2 * (x >> a.u_log2) + (m != 0)) * a.colT_pitch + y;
}
// Store a ring pixel's dwell: image, plus the transposed column copy when x is a column line.
__device__ __forceinline__ void store_ring(const LevelArgs &a, int x, int y, int v)
{
    a.out[(long long)y * a.pitch + x] = v;
    if (a.colT && on_col_line(a, x))
        a.colT[colT_index(a, x, y)] = v;
}

// Per-level-0-tile executed-iteration counter (stats builds only; used by the multi-GPU
// cost-ranked deal's preview run).
__device__ __forceinline__ int tile_of(const LevelArgs &a, int x, int y)
{
    return ((y >> a.d0_log2) << a.g_log2) + (x >> a.d0_log2);
}
__device__ __forceinline__ void add_tile_cost(const LevelArgs &a, int x, int y, int v)
{
    if (a.tile_cost)
        atomicAdd(&a.tile_cost[tile_of(a, x, y)], (unsigned long long)v);
}

// --------------------------------------------------------------------------- PDL
// Programmatic dependent launch (the level chain's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel lets its
// successor launch as soon as all of its blocks are running, then waits for its own
// predecessor's completion (and memory flush) before touching any data, so the successor's
// launch and block scheduling overlap this kernel's tail.  Both are no-ops for a kernel
// launched without the attribute.
__device__ __forceinline__ void pdl_entry()
{
#if MANDEL_PDL
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
// The lane-refill kernels: wait only; they trigger their successor in the tail (refill.cuh
// pdl_trigger, MANDEL_PDL_LATE).
__device__ __forceinline__ void pdl_entry_refill(bool late)
{
#if MANDEL_PDL
    if (!(MANDEL_PDL_LATE && late))
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// The call's region map and maxdwell, read from the device parameter block (written by the
// stream-ordered copy that precedes the graph launch).
__device__ __forceinline__ LevelArgs with_params(LevelArgs a)
{
    a.map = a.prm->map;
    a.maxdwell = a.prm->maxdwell;
    if (a.ntiles < 0) // device tile list: its length was copied into the block by the graph
        a.ntiles = a.prm->ntiles;
    return a;
}

// --------------------------------------------------------------------------- helpers
__device__ __forceinline__ uint32_t level_count(const LevelArgs &a)
{
    // |G_0| = number of tiles; |G_{l}| = r^2 * count_{l-1} ("count")
    if (a.level == 0)
        return (uint32_t)a.ntiles;
    return (uint32_t)(a.r * a.r) * *((volatile uint32_t *)&a.hdr->n_subdiv[a.level - 1]);
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int TPB>
__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v, unsigned long long *s)
{
    v = warp_sum_u64(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0)
        s[w] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < TPB / 32; ++i)
            t += s[i];
    return t; // valid in thread 0
}

// --------------------------------------------------------------------------- Ex
// Exhaustive approach: one thread per pixel over the n x n grid.  K is the
// escape-test interval of the dwell core (dwell.cuh): the plain baseline uses the same K = 8
// as the paper-faithful ASK kernels; the tuned variant (mandel_exhaustive_tuned) tests every
// 32 steps, so the per-chunk bookkeeping (state save, test, branch) costs ~4% of the issue
// slots instead of ~13%, at the price of a longer exact replay once per pixel.
template <int BX, int BY, int K = DWELL_K>
__global__ void __launch_bounds__(BX *BY) k_exhaustive(ExArgs a)
{
    const int x = blockIdx.x * BX + threadIdx.x;
    const int y = blockIdx.y * BY + threadIdx.y;
    if (x >= a.n || y >= a.n)
        return;
    const int v = dwell<K>(pix_re(a.map, x), pix_im(a.map, y), a.maxdwell);
    a.out[(long long)y * a.pitch + x] = v;
}

// --------------------------------------------------------------------------- FP32 probe
// Measured denominator of the ALU roofline (P:280-287 models the machine as q processors of
// c lanes): the dwell step itself (7 non-fused FP32 ops, dwell.cuh) on CH independent orbits
// per thread from a non-escaping c (c = -1: period-2 cycle), no escape test, so the only
// instructions in the loop are the 7 * CH FP32 ops per step.  Ops/s = 7 * CH * steps *
// threads / time.
template <int CH>
__global__ void __launch_bounds__(256) k_probe_fp32(float cr, float ci, int steps, float *sink)
{
    float x[CH], y[CH], x2[CH], y2[CH], c[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
        x[j] = y[j] = x2[j] = y2[j] = 0.0f;
        c[j] = __fadd_rn(cr, __fmul_rn((float)(threadIdx.x * CH + j), 1e-9f));
    }
    for (int i = 0; i < steps; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
#pragma unroll
            for (int j = 0; j < CH; ++j)
                MANDEL_STEP(x[j], y[j], x2[j], y2[j], c[j], ci);
        }
    }
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < CH; ++j)
        acc = __fadd_rn(acc, __fadd_rn(x[j], y[j]));
    if (acc == 12345.0f) // never true; keeps the loop alive
        sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// --------------------------------------------------------------------------- multi-GPU deal
// Graham's longest-processing-time list schedule of the level-0 tiles over `world` ranks
// (the multi-GPU partition of SURVEY.md §8(e); same rule as paper_2206_02255_b200/deal.py
// `lpt`): tiles in descending cost (ties: lower id first), each to the currently least-loaded
// rank (ties: lower rank).  Every rank runs it on the same all-reduced cost vector, so all ranks
// derive the same partition without further communication.  Writes rank `rank`'s tiles in that
// descending order (its level-0 offset list order) and their count.  One block; G <= 4096.
__global__ void __launch_bounds__(1024) k_deal_lpt(const unsigned long long *costs, int G, int world, int rank,
                                                   int32_t *tiles_out, int32_t *ntiles_out)
{
    __shared__ unsigned long long key[4096];
    __shared__ unsigned long long load[64];
    int P = 1;
    while (P < G)
        P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        // descending cost, ascending id: sort keys (cost << 16 | (0xffff - id)) descending;
        // padding entries sort last
        key[i] = i < G ? ((costs[i] & 0xffffffffffffull) << 16) | (unsigned long long)(0xffff - i) : 0ull;
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) // bitonic sort, descending
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const bool desc = (i & k) == 0;
                    const unsigned long long a = key[i], b = key[l];
                    if (desc ? (a < b) : (a > b)) {
                        key[i] = b;
                        key[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    if (threadIdx.x == 0 && world <= 8) { // loads in registers (the usual case)
        unsigned long long l[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            l[q] = q < world ? 0ull : ~0ull;
        int n = 0;
        for (int i = 0; i < G; ++i) {
            const unsigned long long k = key[i];
            const int id = 0xffff - (int)(k & 0xffffull);
            int best = 0;
            unsigned long long bl = l[0];
#pragma unroll
            for (int q = 1; q < 8; ++q)
                if (l[q] < bl) {
                    bl = l[q];
                    best = q;
                }
#pragma unroll
            for (int q = 0; q < 8; ++q)
                l[q] += q == best ? (k >> 16) : 0ull;
            if (best == rank)
                tiles_out[n++] = id;
        }
        *ntiles_out = n;
    } else if (threadIdx.x == 0) {
        for (int q = 0; q < world; ++q)
            load[q] = 0ull;
        int n = 0;
        for (int i = 0; i < G; ++i) {
            const int id = 0xffff - (int)(key[i] & 0xffffull);
            int best = 0;
            for (int q = 1; q < world; ++q)
                if (load[q] < load[best])
                    best = q;
            load[best] += key[i] >> 16;
            if (best == rank)
                tiles_out[n++] = id;
        }
        *ntiles_out = n;
    }
}

// --------------------------------------------------------------------------- init
// Level-0 offset list: the initial g x g split ("initial compute grid |G_0|"),
// canonical order or the caller's tile subset; zero the counters.
__global__ void k_init(LevelArgs a_)
{
    pdl_entry();
    LevelArgs a = with_params(a_);
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (a.src_ntiles) { // device tile list: length and ids straight from the caller's buffers;
        // the length also goes to the parameter block for the later kernels (with_params)
        a.ntiles = *a.src_ntiles;
        a.tiles = a.src_tiles;
        if (t == 0)
            const_cast<DevParams *>(a.prm)->ntiles = a.ntiles;
    }
    if (a.zero_costs && a.tile_cost && t < a.g * a.g)
        a.tile_cost[t] = 0ull;
    constexpr int hdr_words = sizeof(WsHeader) / 4;
    uint32_t *hw = reinterpret_cast<uint32_t *>(a.hdr);
    constexpr int ng_word = (int)(offsetof(WsHeader, ngroups) / 4);
    if (t >= 8 && t < hdr_words)
        hw[t] = (t == ng_word) ? (uint32_t)a.ngroups : 0u;
    if (t == 0) {
        a.hdr->magic = WS_MAGIC;
        a.hdr->levels = (uint32_t)a.levels;
        a.hdr->n = 0; // filled below by thread 1 (keeps t==0 short)
        a.hdr->g = (uint32_t)a.g;
        a.hdr->r = (uint32_t)a.r;
        a.hdr->B = (uint32_t)a.B;
        a.hdr->ntiles = (uint32_t)a.ntiles;
        a.hdr->scheme = (uint32_t)a.scheme;
    }
    if (t == 1)
        a.hdr->n = (uint32_t)(a.d * a.g);
    if (t < a.ntiles) {
        const int k = a.tiles ? a.tiles[t] : t;
        const int gx = k % a.g, gy = k / a.g;
        const_cast<uint32_t *>(a.olt_in)[t] = pack_xy(gx * a.d, gy * a.d);
    }
}

// --------------------------------------------------------------------------- decisions
// Common tail of the per-region decision: uniform -> fill list;
// non-uniform and d/r >= B -> reserve r^2 consecutive OLT slots with one atomicAdd on the
// level's count (compact concurrent insertion, in the region's length bucket); else
// -> leaf list (length bucket).  nmax: ring pixels at maxdwell, ring: ring size.
// Returns the reserved parent slot (or UINT_MAX) to the caller's lane/thread.
// fill_list = false: the caller fills the region itself (ASK-SBR's Delta[T]) and
// only the count is kept.
__device__ __forceinline__ uint32_t decide(const LevelArgs &a, uint32_t off, int lo, int hi, int nmax, int ring,
                                           bool fill_list = true)
{
    if (lo == hi) {
        const uint32_t e = atomicAdd(&a.hdr->n_fill[a.level], 1u);
        if (fill_list)
            a.fill[e] = make_uint2(off, (uint32_t)lo);
        return UINT_MAX;
    }
    const int b = length_bucket(a, hi, nmax, ring);
    if (a.subdivide) {
        atomicAdd(&a.hdr->n_subdiv[a.level], 1u);
        return bucket_put(b, atomicAdd(&a.hdr->n_sub_b[a.level][b], 1u), a.capP);
    }
    atomicAdd(&a.hdr->n_leaf, 1u);
    a.leaf[bucket_put(b, atomicAdd(&a.hdr->n_leaf_b[b], 1u), a.capL)] = off;
    return UINT_MAX;
}

// --------------------------------------------------------------------------- SBR / MBR
// The block of TPB threads that decided region (x0, y0, d) uniform writes v to all its d*d
// pixels (the ring already holds v): 128-bit stores when the rows are 16-byte aligned.
template <int TPB>
__device__ __forceinline__ void block_fill_region(const LevelArgs &a, int x0, int y0, int d, int v, bool vec)
{
    if (vec) {
        const int q = d >> 2; // int4 per row
        const int4 v4 = make_int4(v, v, v, v);
        for (int t = threadIdx.x; t < d * q; t += TPB) {
            const int row = t / q, c = t - row * q;
            __stcs(reinterpret_cast<int4 *>(a.out + (long long)(y0 + row) * a.pitch + x0) + c, v4);
        }
    } else {
        for (int t = threadIdx.x; t < d * d; t += TPB) {
            const int row = t / d, c = t - row * d;
            a.out[(long long)(y0 + row) * a.pitch + x0 + c] = v;
        }
    }
}

// ASK level kernel of the paper's two schemes: one block of TPB
// threads per region (persistent, grid-stride over the level's OLT).  The block's warps
// split the region's 4d-4 border pixels (query Q), write their dwells to the image (they
// are final values), and reduce (min, max) with warp reductions + shared memory; uniform
// iff min == max; thread 0 appends (PS).  FILL (ASK-SBR, Delta[(1-P) T]): the same block
// then fills a uniform region.  !FILL (ASK-MBR, nabla[(1-P) T]): uniform regions go to the
// level's fill list for the flat multi-block k_fill.
template <int TPB, bool STATS, bool FILL = false>
__global__ void __launch_bounds__(TPB) k_sbr_level(LevelArgs a_)
{
    const LevelArgs a = with_params(a_);
    __shared__ int s_lo[TPB / 32], s_hi[TPB / 32], s_nm[TPB / 32];
    __shared__ unsigned long long s_sum[TPB / 32];
    __shared__ uint32_t s_base;
    __shared__ int s_fillv;
    const uint32_t count = level_count(a);
    const int d = a.d, ring = 4 * d - 4, s = d / a.r, rr = a.r * a.r;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const BucketMap bm = sub_buckets(a);
    for (uint32_t ri = blockIdx.x; ri < count; ri += gridDim.x) {
        const uint32_t off = region_origin(a, ri, bm);
        const int x0 = unpack_x(off), y0 = unpack_y(off);
        int lo = INT_MAX, hi = INT_MIN, nm = 0;
        unsigned long long it = 0;
        for (int b = threadIdx.x; b < ring; b += TPB) {
            int x, y;
            ring_pixel(b, d, x0, y0, x, y);
            const int v = dwell<DWELL_K>(pix_re(a.map, x), pix_im(a.map, y), a.maxdwell);
            a.out[(long long)y * a.pitch + x] = v;
            lo = min(lo, v);
            hi = max(hi, v);
            nm += v == a.maxdwell;
            if (STATS) {
                it += (unsigned long long)v;
                add_tile_cost(a, x, y, v);
            }
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        nm = (int)__reduce_add_sync(0xffffffffu, (unsigned)nm);
        if (l == 0) {
            s_lo[w] = lo;
            s_hi[w] = hi;
            s_nm[w] = nm;
        }
        if (STATS)
            it = block_sum_u64<TPB>(it, s_sum);
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int i = 1; i < TPB / 32; ++i) {
                lo = min(lo, s_lo[i]);
                hi = max(hi, s_hi[i]);
                nm += s_nm[i];
            }
            s_base = decide(a, off, lo, hi, nm, ring, !FILL);
            s_fillv = (lo == hi) ? lo : INT_MIN;
            if (STATS) {
                atomicAdd(&a.hdr->border_px[a.level], (unsigned long long)ring);
                atomicAdd(&a.hdr->border_iters[a.level], it);
            }
        }
        __syncthreads();
        const uint32_t base = s_base;
        if (base != UINT_MAX)
            for (int t = threadIdx.x; t < rr; t += TPB)
                a.olt_out[(size_t)base * rr + t] = pack_xy(x0 + (t % a.r) * s, y0 + (t / a.r) * s);
        if (FILL && s_fillv != INT_MIN)
            block_fill_region<TPB>(a, x0, y0, d, s_fillv, a.fill_vec != 0);
        __syncthreads();
    }
}

// Leaf work L, SBR: one block per last-level non-uniform region computes its
// (d-2)^2 interior pixels (the border is already in the image).
template <int TPB, bool STATS>
__global__ void __launch_bounds__(TPB) k_sbr_leaf(LevelArgs a_)
{
    const LevelArgs a = with_params(a_);
    __shared__ unsigned long long s_sum[TPB / 32];
    const uint32_t count = *((volatile uint32_t *)&a.hdr->n_leaf);
    const int d = a.d, m = d - 2, I = m * m;
    const BucketMap lb = leaf_buckets(a);
    for (uint32_t li = blockIdx.x; li < count; li += gridDim.x) {
        const uint32_t off = a.leaf[lb.slot(li)];
        const int x0 = unpack_x(off) + 1, y0 = unpack_y(off) + 1;
        unsigned long long it = 0;
        for (int p = threadIdx.x; p < I; p += TPB) {
            const int x = x0 + p % m, y = y0 + p / m;
            const int v = dwell<DWELL_K>(pix_re(a.map, x), pix_im(a.map, y), a.maxdwell);
            a.out[(long long)y * a.pitch + x] = v;
            if (STATS) {
                it += (unsigned long long)v;
                add_tile_cost(a, x, y, v);
            }
        }
        if (STATS) {
            it = block_sum_u64<TPB>(it, s_sum);
            if (threadIdx.x == 0) {
                atomicAdd(&a.hdr->leaf_px, (unsigned long long)I);
                atomicAdd(&a.hdr->leaf_iters, it);
            }
        }
    }
}

// --------------------------------------------------------------------------- fill
// Terminal work T ("writes a constant value on each data-element"): every uniform
// region of the level is filled with its border dwell.  Flat over all 16-byte vectors of
// all filled regions (grid-stride), streaming 128-bit stores.
template <bool VEC>
__global__ void __launch_bounds__(256) k_fill(LevelArgs a)
{
    const unsigned long long count = *((volatile uint32_t *)&a.hdr->n_fill[a.level]);
    const int d = a.d;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long u = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (VEC) {
        const unsigned long long total = count << a.log2_q4;
        const unsigned long long qmask = (1ull << a.log2_q4) - 1ull;
        const int rmask = (1 << a.log2_row4) - 1;
        for (; u < total; u += stride) {
            const uint2 e = a.fill[u >> a.log2_q4];
            const int rem = (int)(u & qmask);
            const int row = rem >> a.log2_row4, c4 = rem & rmask;
            const int x = unpack_x(e.x) + 4 * c4, y = unpack_y(e.x) + row;
            const int v = (int)e.y;
            __stcs(reinterpret_cast<int4 *>(a.out + (long long)y * a.pitch + x), make_int4(v, v, v, v));
        }
    } else {
        const unsigned long long per = (unsigned long long)d * d;
        const unsigned long long total = count * per;
        for (; u < total; u += stride) {
            const uint2 e = a.fill[u / per];
            const int rem = (int)(u % per);
            const int x = unpack_x(e.x) + rem % d, y = unpack_y(e.x) + rem / d;
            a.out[(long long)y * a.pitch + x] = (int)e.y;
        }
    }
}

// --------------------------------------------------------------------------- B200 scheme
// New border pixels of level `level`, written to the image:
//   level 0: the 4d-4 ring of every level-0 region;
//   level l>0: for every region subdivided at level l-1 (side D = r d), the pixels of its
//   children's rings that are not on its own ring: 2(r-1) full-height internal columns
//   (x0 + k d - 1, x0 + k d; rows y0+1..y0+D-2) and 2(r-1) internal rows without the
//   column pixels (r segments of d-2 pixels each).
// One thread per pixel, flat over all new pixels of the level (grid-stride), so the
// level's whole border work is spread over every SM regardless of region count.
__host__ __device__ __forceinline__ uint32_t new_border_px_per_parent(int D, int r)
{
    const int d = D / r;
    return (uint32_t)(2 * (r - 1) * (D - 2) + 2 * (r - 1) * r * (d - 2));
}

template <bool STATS>
__global__ void __launch_bounds__(256) k_b200_border(LevelArgs a_)
{
    const LevelArgs a = with_params(a_);
    __shared__ unsigned long long s_sum[8];
    unsigned long long total, per;
    const int d = a.d;
    int D = d * a.r; // parent side (level > 0)
    if (a.level == 0) {
        per = (unsigned long long)(4 * d - 4);
        total = per * (unsigned long long)a.ntiles;
    } else {
        per = new_border_px_per_parent(D, a.r);
        total = per * (unsigned long long)(*((volatile uint32_t *)&a.hdr->n_subdiv[a.level - 1]));
    }
    const int rr = a.r * a.r;
    const BucketMap bm = sub_buckets(a);
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long it = 0, px = 0;
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const uint32_t p = (uint32_t)(t / per);
        const int loc = (int)(t - (unsigned long long)p * per);
        int x, y;
        if (a.level == 0) {
            const uint32_t off = a.olt_in[p];
            ring_pixel(loc, d, unpack_x(off), unpack_y(off), x, y);
        } else {
            const uint32_t off = a.olt_in[(size_t)bm.slot(p) * rr]; // first child = parent origin
            const int x0 = unpack_x(off), y0 = unpack_y(off);
            const int pv = 2 * (a.r - 1) * (D - 2);
            if (loc < pv) {
                const int line = loc / (D - 2), row = loc - line * (D - 2);
                x = x0 + (line / 2 + 1) * d - 1 + (line & 1);
                y = y0 + 1 + row;
            } else {
                const int h = loc - pv, seg = d - 2, len = a.r * seg;
                const int line = h / len, c = h - line * len;
                const int k = c / seg, o = c - k * seg;
                y = y0 + (line / 2 + 1) * d - 1 + (line & 1);
                x = x0 + k * d + 1 + o;
            }
        }
        const int v = dwell<DWELL_K>(pix_re(a.map, x), pix_im(a.map, y), a.maxdwell);
        store_ring(a, x, y, v);
        if (STATS) {
            it += (unsigned long long)v;
            px += 1;
            add_tile_cost(a, x, y, v);
        }
    }
    if (STATS) {
        it = block_sum_u64<256>(it, s_sum);
        if (threadIdx.x == 0 && it)
            atomicAdd(&a.hdr->border_iters[a.level], it);
        px = block_sum_u64<256>(px, s_sum);
        if (threadIdx.x == 0 && px)
            atomicAdd(&a.hdr->border_px[a.level], px);
    }
}

// Classification: read each region's 4d-4 ring dwells back (rows from the
// image, columns from colT), reduce (min, max) with warp reductions, decide, and append
// (children written by the region's lanes).  WPR warps per region: half a warp (WPR = 0) or
// one warp for small rings; the whole 256-thread block for large ones (d >= 256, i.e. the
// first levels, where a warp per region would serialise ~d/8 dependent load rounds).
template <int WPR>
__global__ void __launch_bounds__(256) k_b200_classify(LevelArgs a_)
{
    pdl_entry();
    const LevelArgs a = with_params(a_);
    // threads per region: a quarter (WPR = -1) or half a warp (WPR = 0: small rings, more
    // regions in flight per warp at the deep levels), a warp, or WPR warps
    constexpr int TPR = WPR == 0 ? 16 : WPR < 0 ? 8 : 32 * WPR;
    constexpr int RPB = 256 / TPR; // regions per block round
    __shared__ int s_lo[8], s_hi[8], s_nm[8];
    __shared__ uint32_t s_base[RPB];
    const unsigned gmask = TPR == 8    ? 0xffu << (threadIdx.x & 24)
                           : TPR == 16 ? ((threadIdx.x & 16) ? 0xffff0000u : 0x0000ffffu)
                                       : 0xffffffffu;
    const uint32_t count = level_count(a);
    const int d = a.d, ring = 4 * d - 4, s = d / a.r, rr = a.r * a.r;
    const int t = threadIdx.x % TPR, w = threadIdx.x >> 5, slot = threadIdx.x / TPR;
    const uint32_t per_block = 256 / TPR;
    const BucketMap bm = sub_buckets(a);
    for (uint32_t ri0 = blockIdx.x * per_block; ri0 < count; ri0 += gridDim.x * per_block) {
        const uint32_t ri = ri0 + slot;
        const bool valid = ri < count;
        const uint32_t off = valid ? region_origin(a, ri, bm) : 0u;
        const int x0 = unpack_x(off), y0 = unpack_y(off);
        int lo = INT_MAX, hi = INT_MIN, nm = 0; // nm: ring pixels at maxdwell (length bucket)
        if (valid) {
            // batches of 8 independent loads in flight per thread (the ring of a level-0
            // region is 8188 pixels: latency, not bandwidth, bounds this loop)
            for (int b0 = t; b0 < ring; b0 += 8 * TPR) {
                int v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int b = b0 + j * TPR;
                    int x, y;
                    ring_pixel(b < ring ? b : 0, d, x0, y0, x, y);
                    const int *src = (a.colT && b >= 2 * d) ? a.colT + colT_index(a, x, y)
                                                            : a.out + (long long)y * a.pitch + x;
                    v[j] = b < ring ? __ldcg(src) : v[0];
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    lo = min(lo, v[j]);
                    hi = max(hi, v[j]);
                    nm += (b0 + j * TPR < ring) && v[j] == a.maxdwell;
                }
            }
        }
        lo = __reduce_min_sync(gmask, lo);
        hi = __reduce_max_sync(gmask, hi);
        nm = (int)__reduce_add_sync(gmask, (unsigned)nm);
        if (WPR > 1) {
            if ((threadIdx.x & 31) == 0) {
                s_lo[w] = lo;
                s_hi[w] = hi;
                s_nm[w] = nm;
            }
            __syncthreads();
            if (t == 0) {
                for (int k = 1; k < WPR; ++k) {
                    lo = min(lo, s_lo[k]);
                    hi = max(hi, s_hi[k]);
                    nm += s_nm[k];
                }
                s_base[slot] = valid ? decide(a, off, lo, hi, nm, ring) : UINT_MAX;
            }
            __syncthreads();
        } else {
            // Block-aggregated appends: one atomicAdd per outcome per block of 8 or 16 regions
            // instead of two per region (the deep levels hold ~10^5 regions, and per-region
            // atomics on a handful of counters serialise in L2).  Same outcomes and slot
            // addressing as decide(): subdivided parents and leaves by length bucket.
            __shared__ int s_cat[RPB];
            __shared__ uint32_t s_cb[10], s_rank[RPB];
            if (t == 0) {
                int cat = 0; // 0 none, 1 fill, 2+b subdivide (bucket b), 6+b leaf (bucket b)
                if (valid)
                    cat = lo == hi ? 1 : (a.subdivide ? 2 : 6) + length_bucket(a, hi, nm, ring);
                s_cat[slot] = cat;
            }
            __syncthreads();
            if (threadIdx.x < 32) { // warp 0: per-category counts and ranks by ballot (RPB <= 32)
                const int k = threadIdx.x;
                const int cat = k < RPB ? s_cat[k] : 0;
                const unsigned lt = (1u << k) - 1u;
                uint32_t n_mine = 0u; // lane c (1..9): the block's count of category c
                uint32_t rank = 0u;
#pragma unroll
                for (int c = 1; c < 10; ++c) {
                    const unsigned m = __ballot_sync(0xffffffffu, cat == c);
                    if (cat == c)
                        rank = (uint32_t)__popc(m & lt);
                    if (k == c)
                        n_mine = (uint32_t)__popc(m);
                }
                const uint32_t ns = (uint32_t)__popc(__ballot_sync(0xffffffffu, cat >= 2 && cat < 6));
                const uint32_t nl = (uint32_t)__popc(__ballot_sync(0xffffffffu, cat >= 6));
                // every append counter of the round at once, one lane each (all in flight)
                uint32_t b0 = 0u;
                if (n_mine) {
                    unsigned *ctr = k == 1 ? &a.hdr->n_fill[a.level]
                                  : k < 6  ? &a.hdr->n_sub_b[a.level][k - 2]
                                           : &a.hdr->n_leaf_b[k - 6];
                    b0 = atomicAdd(ctr, n_mine);
                }
                if (k == 10 && ns)
                    atomicAdd(&a.hdr->n_subdiv[a.level], ns);
                if (k == 11 && nl)
                    atomicAdd(&a.hdr->n_leaf, nl);
                if (k >= 1 && k < 10)
                    s_cb[k] = b0;
                if (k < RPB)
                    s_rank[k] = rank;
            }
            __syncthreads();
            if (t == 0) {
                const int cat = s_cat[slot];
                const uint32_t e = s_cb[cat] + s_rank[slot];
                uint32_t base = UINT_MAX;
                if (cat == 1)
                    a.fill[e] = make_uint2(off, (uint32_t)lo);
                else if (cat >= 2 && cat < 6)
                    base = bucket_put(cat - 2, e, a.capP);
                else if (cat >= 6)
                    a.leaf[bucket_put(cat - 6, e, a.capL)] = off;
                s_base[slot] = base;
            }
            __syncthreads();
        }
        const uint32_t base = s_base[slot];
        if (base != UINT_MAX)
            for (int c = t; c < rr; c += TPR)
                a.olt_out[(size_t)base * rr + c] = pack_xy(x0 + (c % a.r) * s, y0 + (c / a.r) * s);
        __syncthreads();
    }
}

// Leaf interiors, flat: one thread per interior pixel of all leaves (grid-stride).
template <bool STATS>
__global__ void __launch_bounds__(256) k_b200_leaf(LevelArgs a_)
{
    const LevelArgs a = with_params(a_);
    __shared__ unsigned long long s_sum[8];
    const int d = a.d, m = d - 2;
    const unsigned long long I = (unsigned long long)m * m;
    const unsigned long long total = I * (unsigned long long)(*((volatile uint32_t *)&a.hdr->n_leaf));
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const BucketMap lb = leaf_buckets(a);
    unsigned long long it = 0, px = 0;
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const uint32_t li = (uint32_t)(t / I);
        const int loc = (int)(t - (unsigned long long)li * I);
        const uint32_t off = a.leaf[lb.slot(li)];
        const int x = unpack_x(off) + 1 + loc % m, y = unpack_y(off) + 1 + loc / m;
        const int v = dwell<DWELL_K>(pix_re(a.map, x), pix_im(a.map, y), a.maxdwell);
        a.out[(long long)y * a.pitch + x] = v;
        if (STATS) {
            it += (unsigned long long)v;
            px += 1;
            add_tile_cost(a, x, y, v);
        }
    }
    if (STATS) {
        it = block_sum_u64<256>(it, s_sum);
        if (threadIdx.x == 0 && it)
            atomicAdd(&a.hdr->leaf_iters, it);
        px = block_sum_u64<256>(px, s_sum);
        if (threadIdx.x == 0 && px)
            atomicAdd(&a.hdr->leaf_px, px);
    }
}

// --------------------------------------------------------------------------- lane refill
// B200 border and leaf kernels on the lane-refill engine (refill.cuh): the
// same flat index spaces as k_b200_border / k_b200_leaf, computed by persistent warps whose
// lanes take a new pixel as soon as theirs is done.

// Leaf interiors: t = leaf * (d-2)^2 + row-major interior offset.
struct LeafMap {
    const uint32_t *leaf;
    BucketMap lb;      // leaves in length-bucket order (longest first)
    FastDiv fI, fm;    // I = (d-2)^2, m = d-2
    __device__ __forceinline__ void operator()(uint32_t t, int &x, int &y) const
    {
        const uint32_t li = fdiv(t, fI), loc = t - li * fI.d;
        const uint32_t off = leaf[lb.slot(li)];
        const uint32_t row = fdiv(loc, fm);
        x = unpack_x(off) + 1 + (int)(loc - row * fm.d);
        y = unpack_y(off) + 1 + (int)row;
    }
};

// New border pixels of a level (same enumeration as k_b200_border).
struct BorderMap {
    const uint32_t *olt;
    BucketMap bm;      // parents in length-bucket order (longest first)
    int level, d, r, D;
    FastDiv fper, fcol, fseg, flen; // per, D-2, d-2, r*(d-2)
    __device__ __forceinline__ void operator()(uint32_t t, int &x, int &y) const
    {
        const uint32_t p = fdiv(t, fper), loc = t - p * fper.d;
        if (level == 0) {
            const uint32_t off = olt[p];
            ring_pixel((int)loc, d, unpack_x(off), unpack_y(off), x, y);
            return;
        }
        const uint32_t slot = bm.slot(p);
        const uint32_t off = olt[(size_t)slot * (uint32_t)(r * r)]; // first child = parent origin
        const int x0 = unpack_x(off), y0 = unpack_y(off);
        const uint32_t pv = (uint32_t)(2 * (r - 1)) * fcol.d;
        if (loc < pv) {
            const uint32_t line = fdiv(loc, fcol), row = loc - line * fcol.d;
            x = x0 + ((int)line / 2 + 1) * d - 1 + (int)(line & 1);
            y = y0 + 1 + (int)row;
        } else {
            const uint32_t h = loc - pv;
            const uint32_t line = fdiv(h, flen), c = h - line * flen.d;
            const uint32_t k = fdiv(c, fseg), o = c - k * fseg.d;
            y = y0 + ((int)line / 2 + 1) * d - 1 + (int)(line & 1);
            x = x0 + (int)k * d + 1 + (int)o;
        }
    }
};

// Per-block tile-cost counters in shared memory (MANDEL_FLAG_TILE_COST in the refill kernels):
// a 32-bit low word per tile, updated with native shared atomics, and a carry word bumped
// when the low word wraps (exact for any total); flushed once per block.  A 64-bit shared
// atomicAdd compiles to a CAS spin loop on sm_100 (measured: the counting pass cost 30% more
// than the plain step with it).
constexpr int TC_SMEM = MANDEL_SV_C ? 1008 : 1024; // (SV_C: the leaf kernel stays below 48 KB of static shared memory)
struct TileCostSmem {
    unsigned lo[TC_SMEM], hi[TC_SMEM];
};
template <bool STATS>
struct TcStorage { // the counters only in the STATS instantiation of a kernel
    TileCostSmem t;
    __device__ __forceinline__ TileCostSmem *ptr() { return &t; }
};
template <>
struct TcStorage<false> {
    __device__ __forceinline__ TileCostSmem *ptr() { return nullptr; }
};

// Count modes of the refill kernels: CM_NONE, CM_STATS (per-level pixel/iteration counters
// and exact per-tile costs), CM_SAMPLE (MANDEL_FLAG_TILE_COST_SAMPLED: per-tile costs from
// the pixels on the diagonal lattice (x + y) mod 64 == 0 only, weighted by 64 -- the
// multi-GPU deal's every-step feedback).  CM_SAMPLE adds its samples with global reductions
// straight from the sink: shared counters would need block barriers, and a kernel with
// __syncthreads gets divergence checks around every ballot of the engine (measured: +4% on
// the C3 step even with the counting itself removed).
constexpr int CM_NONE = 0, CM_STATS = 1, CM_SAMPLE = 2;
#ifndef MANDEL_TC_SAMPLE_LOG2
#define MANDEL_TC_SAMPLE_LOG2 6
#endif
constexpr int TC_SAMPLE_LOG2 = MANDEL_TC_SAMPLE_LOG2;
// CM_SAMPLE counts each sampled pixel as its dwell plus TC_PX_COST: the deal balances time,
// and a computed pixel costs the engine's per-pixel work (fetch, park, replay, store) besides
// its iterations.  64 balanced the 8-way deal best in time (max/mean 1.023 -> 1.011 at C3,
// 1.036 -> 1.023 at C4, 1.048 -> 1.007 at C5 against 0; profiles/r02_deal_proxy.jsonl).
#ifndef MANDEL_TC_PX_COST
#define MANDEL_TC_PX_COST 64
#endif
constexpr int TC_PX_COST = MANDEL_TC_PX_COST;

template <int CM, bool RING>
struct StoreSink {
    const LevelArgs *a;
    unsigned long long iters, px;
    TileCostSmem *s_tc; // per-block tile costs in shared memory (NULL: global atomics)
    __device__ __forceinline__ void count_tile(int x, int y, int v)
    {
        if (s_tc) {
            const int t = tile_of(*a, x, y);
            const unsigned old = atomicAdd(&s_tc->lo[t], (unsigned)v);
            if (old + (unsigned)v < old)
                atomicAdd(&s_tc->hi[t], 1u);
        } else {
            add_tile_cost(*a, x, y, v);
        }
    }
    __device__ __forceinline__ void operator()(int x, int y, int v)
    {
        if (RING)
            store_ring(*a, x, y, v);
        else
            a->out[(long long)y * a->pitch + x] = v;
        if (CM == CM_STATS) {
            iters += (unsigned long long)v;
            px += 1;
            count_tile(x, y, v);
        } else if (CM == CM_SAMPLE) { // 1/64 of the pixels: global reductions (no return value)
            if (((x + y) & ((1 << TC_SAMPLE_LOG2) - 1)) == 0)
                atomicAdd(&a->tile_cost[tile_of(*a, x, y)], (unsigned long long)(v + TC_PX_COST) << TC_SAMPLE_LOG2);
        }
    }
};

// MANDEL_FLAG_TILE_COST in the refill kernels: per-pixel atomics on g^2 global counters
// serialise in L2, so a block accumulates them in shared memory (g^2 <= TC_SMEM) and flushes
// once.
__device__ __forceinline__ TileCostSmem *tc_begin(const LevelArgs &a, TileCostSmem *s_tc)
{
    const bool use = a.tile_cost && a.g * a.g <= TC_SMEM;
    if (use)
        for (int i = threadIdx.x; i < a.g * a.g; i += blockDim.x)
            s_tc->lo[i] = s_tc->hi[i] = 0u;
    __syncthreads();
    return use ? s_tc : nullptr;
}
__device__ __forceinline__ void tc_flush(const LevelArgs &a, TileCostSmem *s_tc)
{
    __syncthreads();
    if (s_tc)
        for (int i = threadIdx.x; i < a.g * a.g; i += blockDim.x) {
            const unsigned long long v = ((unsigned long long)s_tc->hi[i] << 32) | s_tc->lo[i];
            if (v)
                atomicAdd(&a.tile_cost[i], v);
        }
}

template <int CM, bool RING>
__device__ __forceinline__ void sink_flush(const StoreSink<CM, RING> &sk, unsigned long long *it_dst,
                                           unsigned long long *px_dst)
{
    if (CM != CM_STATS)
        return;
    __shared__ unsigned long long s_sum[RF_TPB / 32];
    const unsigned long long it = block_sum_u64<RF_TPB>(sk.iters, s_sum);
    if (threadIdx.x == 0 && it)
        atomicAdd(it_dst, it);
    const unsigned long long px = block_sum_u64<RF_TPB>(sk.px, s_sum);
    if (threadIdx.x == 0 && px)
        atomicAdd(px_dst, px);
}

template <int CM>
__global__ void __launch_bounds__(RF_TPB, RFB_MINB) k_b200_border_rf(LevelArgs a_)
{
    pdl_entry_refill(a_.pdl_late != 0);
    const LevelArgs a = with_params(a_);
    __shared__ ParkedPoint s_q[RF_TPB / 32][MANDEL_RFB_PACK ? RF2_QCAP : RF_QCAP];
#if MANDEL_RFB_PACK && MANDEL_RFB_PRE > 0
    __shared__ SvPoint s_sv[RF_TPB / 32][MANDEL_RFB_CH];
#endif
    BorderMap map;
    map.olt = a.olt_in;
    map.bm = sub_buckets(a);
    map.level = a.level;
    map.d = a.d;
    map.r = a.r;
    map.D = a.d * a.r;
    map.fper = a.fd[0];
    map.fcol = a.fd[1];
    map.fseg = a.fd[2];
    map.flen = a.fd[3];
    uint32_t count = (a.level == 0) ? (uint32_t)a.ntiles
                                    : *((volatile uint32_t *)&a.hdr->n_subdiv[a.level - 1]);
    const uint32_t total = map.fper.d * count;
    __shared__ TcStorage<CM == CM_STATS> s_tc; // sampled costs: no shared memory, no block barrier
    StoreSink<CM, true> sink{&a, 0ull, 0ull, CM == CM_STATS ? tc_begin(a, s_tc.ptr()) : nullptr};
#if MANDEL_RFB_PACK && MANDEL_RFB_PRE > 0
    refill_loop2<MANDEL_RFB_K, MANDEL_RFB2_T, MANDEL_RFB_CH, BorderMap, StoreSink<CM, true>, MANDEL_RFB_PRE>(
        a.map, a.maxdwell, total, &a.hdr->cursor[a.level], map, sink, s_q[threadIdx.x >> 5], a.level,
        s_sv[threadIdx.x >> 5]);
#elif MANDEL_RFB_PACK
    refill_loop2<MANDEL_RFB_K, MANDEL_RFB2_T, MANDEL_RFB_CH>(a.map, a.maxdwell, total, &a.hdr->cursor[a.level], map,
                                                             sink, s_q[threadIdx.x >> 5], a.level);
#else
#if MANDEL_RFB_SPRE > 0
    __shared__ SvPoint s_sv[RF_TPB / 32][MANDEL_RFB_CH];
    refill_loop<MANDEL_RFB_K, MANDEL_RFB_T, MANDEL_RFB_CH, BorderMap, StoreSink<CM, true>, MANDEL_RFB_SPRE>(
        a.map, a.maxdwell, total, &a.hdr->cursor[a.level], map, sink, s_q[threadIdx.x >> 5], a.level,
        s_sv[threadIdx.x >> 5]);
#else
    refill_loop<MANDEL_RFB_K, MANDEL_RFB_T, MANDEL_RFB_CH>(a.map, a.maxdwell, total, &a.hdr->cursor[a.level], map,
                                                           sink, s_q[threadIdx.x >> 5], a.level, nullptr,
                                                           a.pdl_late != 0, a.pdl_late ? MANDEL_RFB_CH_DEV : 0u);
#endif
#endif
    if (CM == CM_STATS)
        tc_flush(a, sink.s_tc);
    sink_flush<CM, true>(sink, &a.hdr->border_iters[a.level], &a.hdr->border_px[a.level]);
}

template <int CM>
__global__ void __launch_bounds__(RF_TPB, RFL_MINB) k_b200_leaf_rf(LevelArgs a_)
{
    pdl_entry_refill(a_.pdl_late != 0);
    const LevelArgs a = with_params(a_);
    __shared__ ParkedPoint s_q[RF_TPB / 32][MANDEL_RFL_PACK ? RF2_QCAP : RF_QCAP];
#if MANDEL_RFL_PACK && MANDEL_RFL_PRE > 0
    __shared__ SvPoint s_sv[RF_TPB / 32][MANDEL_RFL_CH];
#endif
    LeafMap map;
    map.leaf = a.leaf;
    map.lb = leaf_buckets(a);
    map.fI = a.fd[0];
    map.fm = a.fd[1];
    const uint32_t total = map.fI.d * *((volatile uint32_t *)&a.hdr->n_leaf);
    __shared__ TcStorage<CM == CM_STATS> s_tc; // sampled costs: no shared memory, no block barrier
    StoreSink<CM, false> sink{&a, 0ull, 0ull, CM == CM_STATS ? tc_begin(a, s_tc.ptr()) : nullptr};
    if (map.fI.d > 0)
#if MANDEL_RFL_PACK
#if MANDEL_RFL_PRE > 0
        refill_loop2<MANDEL_RFL_K, MANDEL_RFL2_T, MANDEL_RFL_CH, LeafMap, StoreSink<CM, false>, MANDEL_RFL_PRE>(
            a.map, a.maxdwell, total, &a.hdr->cursor[MAXL], map, sink, s_q[threadIdx.x >> 5], 15,
            s_sv[threadIdx.x >> 5], a.pdl_late != 0);
#else
        refill_loop2<MANDEL_RFL_K, MANDEL_RFL2_T, MANDEL_RFL_CH>(a.map, a.maxdwell, total, &a.hdr->cursor[MAXL],
                                                                 map, sink, s_q[threadIdx.x >> 5], 15);
#endif
#else
        refill_loop<MANDEL_RFL_K, MANDEL_RFL_T, MANDEL_RFL_CH>(a.map, a.maxdwell, total, &a.hdr->cursor[MAXL], map,
                                                               sink, s_q[threadIdx.x >> 5], 15);
#endif
    if (CM == CM_STATS)
        tc_flush(a, sink.s_tc);
    sink_flush<CM, false>(sink, &a.hdr->leaf_iters, &a.hdr->leaf_px);
}

} // namespace mandel
