// mandel.cu -- C ABI (include/mandel.h): validation, workspace layout, the ASK level loop
// captured once into a CUDA graph per call signature, and launch of the sm_100a kernels.
//
// ASK: one flat kernel per subdivision level, executed serially; the level's
// region count lives in device memory (the OLT "count") and every kernel reads
// it there, so the whole loop -- all levels, fills and leaves -- is one graph launch with
// no host round trip (the paper's host loop copies `count` back after every level).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h> // header-only NVTX v3: ranges cost nothing without a profiler

#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "../../include/mandel.h"
#include "ask_kernels.cuh"

using namespace mandel;

namespace {

// NVTX range for the scope (host side): the API calls, the one-time graph capture +
// instantiation per launch shape, and the bands of the end-to-end call show up by name on an
// Nsight timeline.  (Inside a graph launch the per-level kernels carry their own names.)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

thread_local char g_cuda_err[256] = "";

int cuda_fail(cudaError_t e, const char *what)
{
    snprintf(g_cuda_err, sizeof g_cuda_err, "%s: %s", what, cudaGetErrorString(e));
    return MANDEL_ECUDA;
}

#define CK(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return cuda_fail(e_, #call);                                                       \
    } while (0)

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
int ilog2(int64_t v)
{
    int k = 0;
    while ((int64_t(1) << k) < v)
        ++k;
    return k;
}

bool valid_region(const mandel_region &g)
{
    auto fin = [](double v) { return v == v && v < 1e300 && v > -1e300; };
    return fin(g.re_min) && fin(g.re_max) && fin(g.im_min) && fin(g.im_max) && g.re_min < g.re_max &&
           g.im_min < g.im_max;
}

bool valid_grb(int64_t n, int32_t g, int32_t r, int32_t B)
{
    return is_pow2(n) && n <= 65536 && is_pow2(g) && is_pow2(r) && is_pow2(B) && r >= 2 && B >= 2 &&
           (int64_t)g * B <= n;
}

int levels_of(int64_t n, int32_t g, int32_t r, int32_t B)
{
    int64_t d = n / g;
    int L = 1;
    while (d / r >= B) {
        d /= r;
        ++L;
    }
    return L;
}

// Workspace layout.  cap_l = g^2 r^(2l) (every region may subdivide).
struct Layout {
    int L;
    size_t hdr, prm, prm_bytes, olt[2], fill, leaf, tile_cost, colT, colT_bytes, total;
    int u_log2; // log2 of the leaf side u = (n/g) / r^(L-1)
    size_t fill_off[MAXL]; // element offset of each level's fill segment
    size_t cap[MAXL];
    size_t per_tile[MAXL]; // r^(2l): capacity per level-0 tile at level l
};

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

bool make_layout(int64_t n, int32_t g, int32_t r, int32_t B, Layout &lay)
{
    if (!valid_grb(n, g, r, B))
        return false;
    lay.L = levels_of(n, g, r, B);
    if (lay.L > MAXL)
        return false;
    size_t c = (size_t)g * g, fsum = 0;
    for (int l = 0; l < lay.L; ++l) {
        lay.cap[l] = c;
        lay.per_tile[l] = c / ((size_t)g * g);
        lay.fill_off[l] = fsum;
        fsum += c;
        c *= (size_t)r * r;
    }
    const size_t capmax = lay.cap[lay.L - 1];
    size_t o = 0;
    lay.hdr = o;
    o += (size_t)MAXG * 4096; // one header per group
    // device parameter block (DevParams + the call's tile list), written before every launch
    lay.prm = o;
    lay.prm_bytes = PRM_TILES + (size_t)g * g * 4;
    o = align256(o + lay.prm_bytes);
    // OLT ping-pong and leaf list: two two-ended bucket blocks each (length buckets, §4.8)
    lay.olt[0] = o;
    o = align256(o + 2 * capmax * 4);
    lay.olt[1] = o;
    o = align256(o + 2 * capmax * 4);
    lay.fill = o;
    o = align256(o + fsum * 8);
    lay.leaf = o;
    o = align256(o + 2 * capmax * 4);
    lay.tile_cost = o;
    o = align256(o + (size_t)g * g * 8);
    // transposed column lines (used when the leaf side u >= 8): 2 n/u columns of n rows
    int64_t u = n / g;
    for (int l = 1; l < lay.L; ++l)
        u /= r;
    lay.u_log2 = ilog2(u);
    lay.colT = o;
    lay.colT_bytes = (u >= 8) ? (size_t)(2 * (n / u)) * (size_t)n * 4 : 0;
    o = align256(o + lay.colT_bytes);
    lay.total = o;
    return true;
}

// FastDiv for a divisor that may be 0 (then the map is never evaluated: d.d = 0 marks it).
FastDiv fastdiv_nz(uint32_t d)
{
    if (d == 0) {
        FastDiv f{0u, 0u, 0u, 0u};
        return f;
    }
    return make_fastdiv(d);
}

PixMap make_map(const mandel_region &reg, int64_t n)
{
    PixMap m;
    m.x0 = (float)reg.re_min;
    m.y0 = (float)reg.im_min;
    m.dx = (float)((reg.re_max - reg.re_min) / (double)n);
    m.dy = (float)((reg.im_max - reg.im_min) / (double)n);
    return m;
}

struct DevInfo {
    int sms = 0;
    cudaStream_t cap = nullptr;        // capture origin stream
    cudaStream_t grp[MAXG] = {};       // one capture stream per group chain
    cudaStream_t side[MAXG] = {};      // per group: capture side stream (fill branches)
    cudaEvent_t fork[MAXG] = {};       // per group: fill fork/join event used during capture
    cudaEvent_t start = nullptr, join[MAXG] = {};
    cudaStream_t copy = nullptr;       // mandel_ask_to_host: band copies
    cudaEvent_t band[64] = {}, copied = nullptr;
};

// Graph cache key: everything the captured launches depend on.  The region,
// maxdwell and the tile ids are NOT in it: they live in the workspace's device parameter
// block, rewritten before every launch, so one graph serves every view and tile list.
struct Key {
    int dev;
    int64_t n, pitch;
    int32_t g, r, B, scheme;
    uint32_t flags;
    int32_t *out;
    void *ws;
    size_t ws_bytes;
    int32_t ntiles; // -1: device tile list (length read on the device)
    bool listed;    // an explicit tile list (else canonical 0..g*g-1)
    const void *dtiles, *dntiles; // device tile list and its length (mandel_ask_dtiles), else NULL
    bool operator==(const Key &o) const
    {
        return dev == o.dev && n == o.n && pitch == o.pitch && g == o.g && r == o.r && B == o.B &&
               scheme == o.scheme && flags == o.flags && out == o.out && ws == o.ws && ws_bytes == o.ws_bytes &&
               ntiles == o.ntiles && listed == o.listed && dtiles == o.dtiles && dntiles == o.dntiles;
    }
};

struct Entry {
    Key key;
    cudaGraphExec_t exec = nullptr;
    int ngroups = 1;
    unsigned long long last_use = 0;
    std::vector<cudaEvent_t> evs; // MANDEL_FLAG_TIMING only
    std::vector<int32_t> kinds, t_start, t_end;
    unsigned long long id = 0;
};

std::mutex g_mu;
std::vector<Entry> g_cache;
// Per-device state at stable addresses: a DevInfo pointer stays valid when another device's
// first call grows the table (mandel_ask_to_host keeps one across several calls).
std::vector<std::unique_ptr<DevInfo>> g_dev;
unsigned long long g_clock = 0, g_next_id = 0, g_last_timed = 0;
long long g_captures = 0; // graphs captured so far (mandel_ask_graph_captures)
constexpr size_t kMaxGraphs = 64;
int g_prio_hi = 0, g_prio_lo = 0; // set once by dev_info (cudaDeviceGetStreamPriorityRange)

int dev_info(int dev, DevInfo *&out)
{
    while ((int)g_dev.size() <= dev)
        g_dev.emplace_back(new DevInfo());
    DevInfo &di = *g_dev[dev];
    if (!di.cap) {
        CK(cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev));
        CK(cudaMemcpyToSymbol(c_num_sms, &di.sms, sizeof(int)));
        CK(cudaDeviceGetStreamPriorityRange(&g_prio_lo, &g_prio_hi));
        CK(cudaStreamCreateWithFlags(&di.cap, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&di.start, cudaEventDisableTiming));
        for (int i = 0; i < MAXG; ++i) {
            CK(cudaStreamCreateWithFlags(&di.grp[i], cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&di.side[i], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&di.fork[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&di.join[i], cudaEventDisableTiming));
        }
        CK(cudaStreamCreateWithFlags(&di.copy, cudaStreamNonBlocking));
        for (int i = 0; i < 64; ++i)
            CK(cudaEventCreateWithFlags(&di.band[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&di.copied, cudaEventDisableTiming));
    }
    out = &di;
    return MANDEL_OK;
}

template <typename K>
int resident_grid(K kernel, int tpb, int sms, size_t cap_blocks)
{
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, tpb, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    size_t g = (size_t)per_sm * sms;
    if (cap_blocks < g)
        g = cap_blocks;
    return (int)(g < 1 ? 1 : g);
}

// Classification uses half a warp per region for region sides up to this (ring <= 252 pixels).
#ifndef MANDEL_CLASSIFY_BLOCK_D // classification: a whole block per region from this side up
#define MANDEL_CLASSIFY_BLOCK_D 512 // (round 2, before the ballot appends: 256: C3 7.74 ms, 512: 7.71, 1024: 7.69,
                                    // profiles/r02_ab_classify_block.jsonl; with them 512 is 0.2-0.7% faster
                                    // at C3, C5, C3r8d and C4r8d, 0.15% slower at C4;
                                    // profiles/r02_ab_classify_block_d_final.jsonl)
#endif
#ifndef MANDEL_CLASSIFY_HALF_D
#define MANDEL_CLASSIFY_HALF_D 64
#endif
// ... and a quarter of a warp for sides up to this (ring <= 124 pixels; 0: never).
#ifndef MANDEL_CLASSIFY_QUARTER_D
#define MANDEL_CLASSIFY_QUARTER_D 32
#endif

// Block-scheduling priorities (MANDEL_PRIO): the level chain (border, classification, leaf)
// at the device's greatest priority, the overlapped fills at the least; the graph is
// instantiated with cudaGraphInstantiateFlagUseNodePriority so the per-node priorities apply
// (without that flag the captured priorities are ignored).  An overlapped fill grid otherwise
// takes the SM slots a border kernel frees and the next level's classification waits behind it
// (refill trace: 67-167 us between C3 levels against 12-87 us of classification):
// C3 7.71 -> 7.63 ms, C5 21.02 -> 20.86, C4 32.07 -> 31.51 (profiles/r02_ab_prio_fills.jsonl).
#ifndef MANDEL_PRIO
#define MANDEL_PRIO 1
#endif

// Launch on `s` with programmatic stream serialization (PDL, see pdl_entry()): under stream
// capture this becomes a programmatic edge to the previous kernel node on `s`.
template <typename... KArgs>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, cudaStream_t s, LevelArgs a)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = MANDEL_PDL ? 1 : 0;
    at[1].id = cudaLaunchAttributePriority;
    at[1].val.priority = g_prio_hi;
    cfg.attrs = at;
    cfg.numAttrs = MANDEL_PRIO ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, a);
}

// A fill kernel at the least priority (MANDEL_PRIO), else a plain launch.
template <typename... KArgs>
cudaError_t launch_fill(void (*kernel)(KArgs...), int grid, int block, cudaStream_t s, LevelArgs a)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = g_prio_lo;
    cfg.attrs = at;
    cfg.numAttrs = MANDEL_PRIO ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, a);
}

// Per-kernel timing inside the graph (MANDEL_FLAG_TIMING): an external event-record node
// on the kernel's own stream right before and right after every kernel.
struct Timing {
    bool on = false;
    bool leaf_only = false; // MANDEL_FLAG_TIMING_LEAF: events around the leaf kernel only
    bool next_leaf = false; // set by TBEGIN_LEAF for the next t_begin
    std::vector<cudaEvent_t> evs;        // all events (owned by the cache entry)
    std::vector<int32_t> start, end;     // per kernel: indices into evs
    std::vector<int32_t> kinds;          // per kernel: kind * 100 + level
    int32_t open = -1;
};

int t_begin(Timing *tm, cudaStream_t st)
{
    const bool leaf = tm && tm->next_leaf;
    if (tm)
        tm->next_leaf = false;
    if (!tm || !tm->on || (tm->leaf_only && !leaf)) {
        if (tm)
            tm->open = -1;
        return MANDEL_OK;
    }
    cudaEvent_t ev;
    CK(cudaEventCreate(&ev));
    tm->open = (int32_t)tm->evs.size();
    tm->evs.push_back(ev);
    CK(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal));
    return MANDEL_OK;
}

int t_end(Timing *tm, int kind, int level, cudaStream_t st)
{
    if (!tm || !tm->on || tm->open < 0)
        return MANDEL_OK;
    cudaEvent_t ev;
    CK(cudaEventCreate(&ev));
    tm->start.push_back(tm->open);
    tm->end.push_back((int32_t)tm->evs.size());
    tm->kinds.push_back(kind * 100 + level);
    tm->evs.push_back(ev);
    CK(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal));
    return MANDEL_OK;
}

#define TBEGIN(st)                                                                             \
    do {                                                                                       \
        int m_ = t_begin(tm, (st));                                                            \
        if (m_)                                                                                \
            return m_;                                                                         \
    } while (0)
#define TBEGIN_LEAF(st)                                                                        \
    do {                                                                                       \
        if (tm)                                                                                \
            tm->next_leaf = true;                                                              \
        TBEGIN(st);                                                                            \
    } while (0)
#define TEND(kind, level, st)                                                                  \
    do {                                                                                       \
        int m_ = t_end(tm, (kind), (level), (st));                                             \
        if (m_)                                                                                \
            return m_;                                                                         \
    } while (0)

// One independent ASK chain over a subset of the level-0 tiles: its own
// header, and slices of the OLT / fill / leaf buffers sized for its tiles.
struct Group {
    size_t hdr;               // byte offset of its header
    size_t unit0;             // level-0 tiles of the groups before it (slice offset unit)
    int ntiles;               // -1: device tile list, length in the parameter block
    const int32_t *tiles;     // device-visible tile ids (NULL: canonical 0..ntiles-1)
    int cap_tiles;            // upper bound of ntiles (buffer slices, grid sizes)
};

// Enqueue one group's whole ASK chain on `s` (called under stream capture).
// Fills (HBM-bound) run on the side stream s2 as graph branches forked after each level's
// classification and joined at the end, overlapping the ALU-bound dwell kernels; a fill
// writes only the interior of regions that are terminal, which no later kernel reads.
int enqueue_ask(const Key &k, const Layout &lay, const Group &grp, int ngroups, int sms, cudaStream_t s,
                cudaStream_t s2, cudaEvent_t fork, Timing *tm)
{
    const int ntiles = grp.cap_tiles; // capacities and grid sizes (== grp.ntiles for host lists)
    const size_t Lm = (size_t)lay.L - 1;
    // (ASK-SBR has no fill kernels: nothing to overlap)
    const bool overlap = (k.flags & MANDEL_FLAG_SERIAL) == 0 && k.scheme != MANDEL_SCHEME_SBR;
    cudaStream_t sf = overlap ? s2 : s; // stream of the fill kernels
    char *ws = (char *)k.ws;
    LevelArgs a;
    memset(&a, 0, sizeof a);
    a.prm = (const DevParams *)(ws + lay.prm); // region map + maxdwell: read at kernel entry
    a.pitch = k.pitch;
    a.out = k.out;
    a.hdr = (WsHeader *)(ws + grp.hdr);
    a.leaf = (uint32_t *)(ws + lay.leaf) + 2 * grp.unit0 * lay.per_tile[Lm];
    a.tiles = grp.tiles;
    a.ngroups = ngroups;
    a.r = k.r;
    a.B = k.B;
    a.g = k.g;
    a.ntiles = grp.ntiles;
    a.levels = lay.L;
    a.scheme = k.scheme;
    a.d0 = (int)(k.n / k.g);
    a.d0_log2 = ilog2(k.n / k.g);
    a.g_log2 = ilog2(k.g);
    a.capL = (uint32_t)((size_t)ntiles * lay.per_tile[Lm]);
    a.capP = (uint32_t)((size_t)ntiles * lay.per_tile[Lm] / ((size_t)k.r * k.r));
    a.tile_cost = (k.flags & (MANDEL_FLAG_TILE_COST | MANDEL_FLAG_TILE_COST_SAMPLED))
                      ? (unsigned long long *)(ws + lay.tile_cost)
                      : nullptr;
    const bool stats = (k.flags & (MANDEL_FLAG_STATS | MANDEL_FLAG_TILE_COST)) != 0;
    // refill kernels' count mode (SAMPLED reaches here only for the B200 refill path)
    const int cm = stats ? CM_STATS : (k.flags & MANDEL_FLAG_TILE_COST_SAMPLED) ? CM_SAMPLE : CM_NONE;
    const bool flat = (k.flags & MANDEL_FLAG_FLAT) != 0;
    a.pdl_late = k.dtiles != nullptr; // refill.cuh pdl_trigger
    if (k.scheme == MANDEL_SCHEME_B200 && lay.colT_bytes) {
        a.colT = (int *)(ws + lay.colT);
        a.u_log2 = lay.u_log2;
        a.colT_pitch = k.n;
    }
    const bool vec_ok = ((uintptr_t)k.out % 16 == 0) && (k.pitch % 4 == 0);
    const int d0 = (int)(k.n / k.g);

    // init: level-0 OLT + zeroed counters
    a.level = 0;
    a.d = d0;
    uint32_t *olt_g[2] = {(uint32_t *)(ws + lay.olt[0]) + 2 * grp.unit0 * lay.per_tile[Lm],
                          (uint32_t *)(ws + lay.olt[1]) + 2 * grp.unit0 * lay.per_tile[Lm]};
    a.olt_in = olt_g[0];
    {
        if (ngroups == 1 && k.dtiles) { // device list: k_init copies it (no memcpy graph nodes)
            a.src_tiles = (const int32_t *)k.dtiles;
            a.src_ntiles = (const int32_t *)k.dntiles;
        }
        a.zero_costs = ngroups == 1; // else a memset node before the group branches
        int nthr = ntiles > 1024 ? ntiles : 1024;
        nthr = nthr > k.g * k.g ? nthr : k.g * k.g;
        TBEGIN(s);
        k_init<<<(nthr + 255) / 256, 256, 0, s>>>(a);
        CK(cudaGetLastError());
        TEND(MANDEL_KIND_INIT, 0, s);
    }
    int d = d0;
    for (int l = 0; l < lay.L; ++l) {
        a.level = l;
        a.d = d;
        a.subdivide = (d / k.r >= k.B) ? 1 : 0;
        a.olt_in = olt_g[l & 1];
        a.olt_out = olt_g[(l + 1) & 1];
        a.fill = (uint2 *)(ws + lay.fill) + lay.fill_off[l] + grp.unit0 * lay.per_tile[l];
        // max regions at this level for this call
        size_t cap = (size_t)ntiles;
        for (int i = 0; i < l; ++i)
            cap *= (size_t)k.r * k.r;
        const bool paper = k.scheme == MANDEL_SCHEME_SBR || k.scheme == MANDEL_SCHEME_MBR;
        const bool sbr_fill = k.scheme == MANDEL_SCHEME_SBR; // Delta[T]: the level kernel fills
        a.fill_vec = (vec_ok && d % 4 == 0) ? 1 : 0;
        if (paper) {
            const int ring = 4 * d - 4;
#define SBR_LAUNCH(TPB)                                                                        \
    do {                                                                                       \
        if (sbr_fill) {                                                                        \
            if (stats) {                                                                       \
                int gsz = resident_grid(k_sbr_level<TPB, true, true>, TPB, sms, cap);          \
                k_sbr_level<TPB, true, true><<<gsz, TPB, 0, s>>>(a);                            \
            } else {                                                                           \
                int gsz = resident_grid(k_sbr_level<TPB, false, true>, TPB, sms, cap);         \
                k_sbr_level<TPB, false, true><<<gsz, TPB, 0, s>>>(a);                           \
            }                                                                                  \
        } else if (stats) {                                                                    \
            int gsz = resident_grid(k_sbr_level<TPB, true>, TPB, sms, cap);                    \
            k_sbr_level<TPB, true><<<gsz, TPB, 0, s>>>(a);                                      \
        } else {                                                                               \
            int gsz = resident_grid(k_sbr_level<TPB, false>, TPB, sms, cap);                   \
            k_sbr_level<TPB, false><<<gsz, TPB, 0, s>>>(a);                                     \
        }                                                                                      \
    } while (0)
            TBEGIN(s);
            if (ring >= 256)
                SBR_LAUNCH(256);
            else if (ring >= 128)
                SBR_LAUNCH(128);
            else if (ring >= 64)
                SBR_LAUNCH(64);
            else
                SBR_LAUNCH(32);
#undef SBR_LAUNCH
            CK(cudaGetLastError());
            TEND(MANDEL_KIND_SBR_LEVEL, l, s);
        } else {
            size_t work = (l == 0) ? cap * (size_t)(4 * d - 4)
                                   : (cap / ((size_t)k.r * k.r)) * new_border_px_per_parent(d * k.r, k.r);
            size_t blocks = (work + 255) / 256;
            TBEGIN(s);
            if (flat) {
                if (stats) {
                    int gsz = resident_grid(k_b200_border<true>, 256, sms, blocks);
                    k_b200_border<true><<<gsz, 256, 0, s>>>(a);
                } else {
                    int gsz = resident_grid(k_b200_border<false>, 256, sms, blocks);
                    k_b200_border<false><<<gsz, 256, 0, s>>>(a);
                }
            } else { // lane refill: persistent warps, one per 32 pixels of work at most
                const size_t rf_blocks = (work + RF_TPB - 1) / RF_TPB;
                const uint32_t per = (l == 0) ? (uint32_t)(4 * d - 4) : new_border_px_per_parent(d * k.r, k.r);
                a.fd[0] = fastdiv_nz(per);
                a.fd[1] = fastdiv_nz((uint32_t)(d * k.r - 2));
                a.fd[2] = fastdiv_nz((uint32_t)(d - 2));
                a.fd[3] = fastdiv_nz((uint32_t)(k.r * (d - 2)));
                if (cm == CM_STATS) {
                    int gsz = resident_grid(k_b200_border_rf<CM_STATS>, RF_TPB, sms, rf_blocks);
                    CK(launch_pdl(k_b200_border_rf<CM_STATS>, gsz, RF_TPB, s, a));
                } else if (cm == CM_SAMPLE) {
                    int gsz = resident_grid(k_b200_border_rf<CM_SAMPLE>, RF_TPB, sms, rf_blocks);
                    CK(launch_pdl(k_b200_border_rf<CM_SAMPLE>, gsz, RF_TPB, s, a));
                } else {
                    int gsz = resident_grid(k_b200_border_rf<CM_NONE>, RF_TPB, sms, rf_blocks);
                    CK(launch_pdl(k_b200_border_rf<CM_NONE>, gsz, RF_TPB, s, a));
                }
            }
            CK(cudaGetLastError());
            TEND(MANDEL_KIND_B200_BORDER, l, s);
            TBEGIN(s);
            if (d >= MANDEL_CLASSIFY_BLOCK_D) { // a whole block per region
                int gsz = resident_grid(k_b200_classify<8>, 256, sms, cap);
                CK(launch_pdl(k_b200_classify<8>, gsz, 256, s, a));
            } else if (d <= MANDEL_CLASSIFY_QUARTER_D) { // a quarter of a warp per region
                int gsz = resident_grid(k_b200_classify<-1>, 256, sms, (cap + 31) / 32);
                CK(launch_pdl(k_b200_classify<-1>, gsz, 256, s, a));
            } else if (d <= MANDEL_CLASSIFY_HALF_D) { // half a warp per region
                int gsz = resident_grid(k_b200_classify<0>, 256, sms, (cap + 15) / 16);
                CK(launch_pdl(k_b200_classify<0>, gsz, 256, s, a));
            } else {
                int gsz = resident_grid(k_b200_classify<1>, 256, sms, (cap + 7) / 8);
                CK(launch_pdl(k_b200_classify<1>, gsz, 256, s, a));
            }
            CK(cudaGetLastError());
            TEND(MANDEL_KIND_B200_CLASSIFY, l, s);
        }
        // fill (terminal work) of this level's uniform regions: flat over all of them
        // (B200, MBR); ASK-SBR filled them inside its level kernel
        if (!sbr_fill) {
            const bool vec = vec_ok && d >= 4;
            a.log2_q4 = vec ? ilog2((int64_t)d * d / 4) : 0;
            a.log2_row4 = vec ? ilog2(d / 4) : 0;
            size_t work = cap * (size_t)d * d / (vec ? 4 : 1);
            size_t blocks = (work + 255) / 256;
            if (overlap) { // fork: the fill of level l waits only for its classification
                CK(cudaEventRecord(fork, s));
                CK(cudaStreamWaitEvent(sf, fork, 0));
            }
            TBEGIN(sf);
            if (vec) {
                int gsz = resident_grid(k_fill<true>, 256, sms, blocks);
                CK(launch_fill(k_fill<true>, gsz, 256, sf, a));
            } else {
                int gsz = resident_grid(k_fill<false>, 256, sms, blocks);
                CK(launch_fill(k_fill<false>, gsz, 256, sf, a));
            }
            CK(cudaGetLastError());
            TEND(MANDEL_KIND_FILL, l, sf);
        }
        if (l + 1 < lay.L)
            d /= k.r;
    }
    // leaves of the last level
    {
        a.level = lay.L - 1;
        a.d = d;
        size_t cap = (size_t)ntiles;
        for (int i = 0; i < lay.L - 1; ++i)
            cap *= (size_t)k.r * k.r;
        TBEGIN_LEAF(s);
        if (k.scheme == MANDEL_SCHEME_MBR) { // nabla[L]: multiple blocks per leaf, flat
            size_t blocks = (cap * (size_t)(d - 2) * (d - 2) + 255) / 256;
            if (stats) {
                int gsz = resident_grid(k_b200_leaf<true>, 256, sms, blocks);
                k_b200_leaf<true><<<gsz, 256, 0, s>>>(a);
            } else {
                int gsz = resident_grid(k_b200_leaf<false>, 256, sms, blocks);
                k_b200_leaf<false><<<gsz, 256, 0, s>>>(a);
            }
        } else if (k.scheme == MANDEL_SCHEME_SBR) {
            const int I = (d - 2) * (d - 2);
#define LEAF_LAUNCH(TPB)                                                                       \
    do {                                                                                       \
        if (stats) {                                                                           \
            int gsz = resident_grid(k_sbr_leaf<TPB, true>, TPB, sms, cap);                     \
            k_sbr_leaf<TPB, true><<<gsz, TPB, 0, s>>>(a);                                       \
        } else {                                                                               \
            int gsz = resident_grid(k_sbr_leaf<TPB, false>, TPB, sms, cap);                    \
            k_sbr_leaf<TPB, false><<<gsz, TPB, 0, s>>>(a);                                      \
        }                                                                                      \
    } while (0)
            if (I >= 256)
                LEAF_LAUNCH(256);
            else if (I >= 128)
                LEAF_LAUNCH(128);
            else if (I >= 64)
                LEAF_LAUNCH(64);
            else
                LEAF_LAUNCH(32);
#undef LEAF_LAUNCH
        } else {
            size_t blocks = (cap * (size_t)(d - 2) * (d - 2) + 255) / 256;
            if (flat) {
                if (stats) {
                    int gsz = resident_grid(k_b200_leaf<true>, 256, sms, blocks);
                    k_b200_leaf<true><<<gsz, 256, 0, s>>>(a);
                } else {
                    int gsz = resident_grid(k_b200_leaf<false>, 256, sms, blocks);
                    k_b200_leaf<false><<<gsz, 256, 0, s>>>(a);
                }
            } else {
                a.fd[0] = fastdiv_nz((uint32_t)((d - 2) * (d - 2)));
                a.fd[1] = fastdiv_nz((uint32_t)(d - 2));
                if (cm == CM_STATS) {
                    int gsz = resident_grid(k_b200_leaf_rf<CM_STATS>, RF_TPB, sms, blocks * (256 / RF_TPB));
                    CK(launch_pdl(k_b200_leaf_rf<CM_STATS>, gsz, RF_TPB, s, a));
                } else if (cm == CM_SAMPLE) {
                    int gsz = resident_grid(k_b200_leaf_rf<CM_SAMPLE>, RF_TPB, sms, blocks * (256 / RF_TPB));
                    CK(launch_pdl(k_b200_leaf_rf<CM_SAMPLE>, gsz, RF_TPB, s, a));
                } else {
                    int gsz = resident_grid(k_b200_leaf_rf<CM_NONE>, RF_TPB, sms, blocks * (256 / RF_TPB));
                    CK(launch_pdl(k_b200_leaf_rf<CM_NONE>, gsz, RF_TPB, s, a));
                }
            }
        }
        CK(cudaGetLastError());
        TEND(k.scheme == MANDEL_SCHEME_SBR   ? MANDEL_KIND_SBR_LEAF
             : k.scheme == MANDEL_SCHEME_MBR ? MANDEL_KIND_MBR_LEAF
                                             : MANDEL_KIND_B200_LEAF,
             lay.L - 1, s);
    }
    if (overlap) { // join the fill branches
        CK(cudaEventRecord(fork, sf));
        CK(cudaStreamWaitEvent(s, fork, 0));
    }
    return MANDEL_OK;
}

void free_entry(Entry &e)
{
    if (e.exec)
        cudaGraphExecDestroy(e.exec);
    for (auto ev : e.evs)
        cudaEventDestroy(ev);
    e.evs.clear();
    e.exec = nullptr;
}

int validate_common(const mandel_region &reg, int64_t n, int32_t maxdwell, int32_t *d_out, int64_t pitch)
{
    if (!valid_region(reg) || !is_pow2(n) || n > 65536 || maxdwell < 1 || !d_out || pitch < n)
        return MANDEL_EINVAL;
    return MANDEL_OK;
}

template <int BX, int BY, int K>
int launch_exhaustive(const mandel_region &reg, int64_t n, int32_t maxdwell, int32_t *d_out, int64_t out_pitch,
                      void *stream)
{
    ExArgs a;
    a.map = make_map(reg, n);
    a.n = (int)n;
    a.maxdwell = maxdwell;
    a.pitch = out_pitch;
    a.out = d_out;
    dim3 grid((unsigned)((n + BX - 1) / BX), (unsigned)((n + BY - 1) / BY));
    k_exhaustive<BX, BY, K><<<grid, dim3(BX, BY), 0, (cudaStream_t)stream>>>(a);
    CK(cudaGetLastError());
    return MANDEL_OK;
}
} // namespace

extern "C" {

size_t mandel_ask_workspace_bytes(int64_t n, int32_t g, int32_t r, int32_t B)
{
    Layout lay;
    if (!make_layout(n, g, r, B, lay))
        return 0;
    return lay.total;
}

int32_t mandel_ask_levels(int64_t n, int32_t g, int32_t r, int32_t B)
{
    if (!valid_grb(n, g, r, B))
        return 0;
    return levels_of(n, g, r, B);
}

int mandel_fp32_peak_probe(int32_t steps, double *tops, void *stream)
{
    if (steps < 1 || !tops)
        return MANDEL_EINVAL;
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cudaStream_t st = (cudaStream_t)stream;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = sms * 8; // 8 x 256 threads per SM: 16 warps per sub-partition
    double best = 0.0;
    int rc = MANDEL_OK;
    for (int rep = 0; rep < 4 && rc == MANDEL_OK; ++rep) {
        float ms = 0.0f;
        cudaEventRecord(e0, st);
        k_probe_fp32<2><<<blocks, 256, 0, st>>>(-1.0f, 0.0f, steps, nullptr);
        cudaEventRecord(e1, st);
        cudaError_t e = cudaEventSynchronize(e1);
        if (e == cudaSuccess)
            e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cudaEventElapsedTime(&ms, e0, e1);
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "mandel_fp32_peak_probe");
            break;
        }
        const double ops = 6.0 * 2 * 8 * (double)steps * blocks * 256; // 6 FP32 instructions per step (R4')
        if (rep > 0 && ms > 0.0f && ops / (ms * 1e9) > best) // rep 0 warms up
            best = ops / (ms * 1e9);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *tops = best;
    return rc;
}

int32_t mandel_ask_kernel_count(int64_t n, int32_t g, int32_t r, int32_t B, int32_t scheme)
{
    if (!valid_grb(n, g, r, B))
        return 0;
    const int L = levels_of(n, g, r, B);
    return 1 + L * (scheme == MANDEL_SCHEME_SBR ? 1 : scheme == MANDEL_SCHEME_MBR ? 2 : 3) + 1;
}

long long mandel_ask_graph_captures(void)
{
    std::lock_guard<std::mutex> lk(g_mu);
    return g_captures;
}

int mandel_exhaustive(mandel_region reg, int64_t n, int32_t maxdwell, int32_t *d_out, int64_t out_pitch,
                      void *stream)
{
    int rc = validate_common(reg, n, maxdwell, d_out, out_pitch);
    if (rc)
        return rc;
    // block shape of the flat Ex kernel (tuned on the box like the paper's Table 2 search,
    // P:459-468; profiles/r01_tune_ex.txt)
    return launch_exhaustive<16, 16, DWELL_K>(reg, n, maxdwell, d_out, out_pitch, stream);
}

int mandel_exhaustive_tuned(mandel_region reg, int64_t n, int32_t maxdwell, int32_t *d_out, int64_t out_pitch,
                            void *stream)
{
    int rc = validate_common(reg, n, maxdwell, d_out, out_pitch);
    if (rc)
        return rc;
#ifndef MANDEL_EXT_K
#define MANDEL_EXT_K 32
#endif
    return launch_exhaustive<32, 8, MANDEL_EXT_K>(reg, n, maxdwell, d_out, out_pitch, stream);
}

} // extern "C"

namespace {
// mandel_ask_tiles (host tile list h_tile_ids) and mandel_ask_dtiles (device tile list d_tiles
// of length *d_ntiles, copied into the parameter block by the graph itself).
int ask_launch(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B,
               const int32_t *h_tile_ids, int32_t n_tiles, const int32_t *d_tiles_in, const int32_t *d_ntiles,
               int32_t scheme, uint32_t flags, int32_t *d_out, int64_t out_pitch, void *d_ws, size_t ws_bytes,
               void *stream)
{
    NvtxRange nv(d_tiles_in ? "mandel_ask_dtiles" : "mandel_ask_tiles");
    const bool dlist = d_tiles_in != nullptr;
    int rc = validate_common(reg, n, maxdwell, d_out, out_pitch);
    if (rc)
        return rc;
    if (!valid_grb(n, g, r, B) || !d_ws ||
        (scheme != MANDEL_SCHEME_SBR && scheme != MANDEL_SCHEME_B200 && scheme != MANDEL_SCHEME_MBR) ||
        (flags & ~(MANDEL_FLAG_STATS | MANDEL_FLAG_TIMING | MANDEL_FLAG_TILE_COST | MANDEL_FLAG_FLAT |
                   MANDEL_FLAG_SERIAL | MANDEL_FLAG_GROUPS_MASK | MANDEL_FLAG_TIMING_LEAF |
                   MANDEL_FLAG_TILE_COST_SAMPLED)) != 0 ||
        MANDEL_FLAG_GROUPS_OF(flags) > MAXG)
        return MANDEL_EINVAL;
    // sampled costs exist only in the B200 refill kernels; elsewhere (and next to the exact
    // counters) the call counts exactly
    if ((flags & MANDEL_FLAG_TILE_COST_SAMPLED) &&
        (scheme != MANDEL_SCHEME_B200 || (flags & (MANDEL_FLAG_FLAT | MANDEL_FLAG_STATS | MANDEL_FLAG_TILE_COST))))
        flags = (flags & ~MANDEL_FLAG_TILE_COST_SAMPLED) | MANDEL_FLAG_TILE_COST;
    Layout lay;
    if (!make_layout(n, g, r, B, lay))
        return MANDEL_EINVAL;
    if (ws_bytes < lay.total)
        return MANDEL_EWORKSPACE;
    if ((uintptr_t)d_ws % 256 != 0)
        return MANDEL_EINVAL;
    const int64_t G = (int64_t)g * g;
    if (dlist && (!d_ntiles || h_tile_ids || MANDEL_FLAG_GROUPS_OF(flags) != 1 || G > 4096))
        return MANDEL_EINVAL;
    if (h_tile_ids) {
        if (n_tiles < 0 || n_tiles > G)
            return MANDEL_EINVAL;
        std::vector<char> seen((size_t)G, 0);
        for (int32_t i = 0; i < n_tiles; ++i) {
            const int32_t t = h_tile_ids[i];
            if (t < 0 || t >= G || seen[(size_t)t])
                return MANDEL_EINVAL;
            seen[(size_t)t] = 1;
        }
    } else if (n_tiles != 0) {
        return MANDEL_EINVAL;
    }
    const int ntiles = dlist ? -1 : h_tile_ids ? n_tiles : (int)G;
    const int cap_tiles = dlist ? (int)G : ntiles;
    // groups: the tiles are dealt round-robin in the given order (LPT order is preserved)
    int ngroups = MANDEL_FLAG_GROUPS_OF(flags);
    if (ngroups > cap_tiles)
        ngroups = cap_tiles > 0 ? cap_tiles : 1;
    const bool listed = dlist || h_tile_ids != nullptr || ngroups > 1;

    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_mu);
    DevInfo *di = nullptr;
    if ((rc = dev_info(dev, di)))
        return rc;

    // ---- per-call device parameter block: region map, maxdwell, the group-dealt tile list.
    // Pageable source: cudaMemcpyAsync stages it before returning, so the buffer is free for
    // the next call while this one is still queued.
    thread_local std::vector<unsigned char> hp;
    hp.assign(dlist ? PRM_HOST_BYTES_DTILES : PRM_TILES + (listed ? (size_t)ntiles * 4 : 0), 0);
    DevParams prm;
    memset(&prm, 0, sizeof prm);
    prm.map = make_map(reg, n);
    prm.maxdwell = maxdwell;
    prm.ntiles = ntiles;
    prm.magic = PRM_MAGIC;
    memcpy(hp.data(), &prm, dlist ? PRM_HOST_BYTES_DTILES : sizeof prm);
    std::vector<int> gcount((size_t)ngroups, 0);
    if (!dlist) {
        int32_t *ord = (int32_t *)(hp.data() + PRM_TILES);
        size_t o = 0;
        for (int gi = 0; gi < ngroups; ++gi)
            for (int i = gi; i < ntiles; i += ngroups) {
                if (listed)
                    ord[o++] = h_tile_ids ? h_tile_ids[i] : i;
                ++gcount[(size_t)gi];
            }
    }
    CK(cudaMemcpyAsync((char *)d_ws + lay.prm, hp.data(), hp.size(), cudaMemcpyHostToDevice, (cudaStream_t)stream));

    Key key{dev, n, out_pitch, g, r, B, scheme, flags, d_out, d_ws, ws_bytes, ntiles, listed, d_tiles_in, d_ntiles};
    Entry *hit = nullptr;
    for (auto &e : g_cache)
        if (e.key == key) {
            hit = &e;
            break;
        }
    if (!hit) {
        if (g_cache.size() >= kMaxGraphs) { // evict least recently used
            size_t lru = 0;
            for (size_t i = 1; i < g_cache.size(); ++i)
                if (g_cache[i].last_use < g_cache[lru].last_use)
                    lru = i;
            free_entry(g_cache[lru]);
            g_cache.erase(g_cache.begin() + (long)lru);
        }
        NvtxRange nv_cap("capture + instantiate (new launch shape)");
        Entry e;
        e.key = key;
        e.ngroups = ngroups;
        const int32_t *d_tiles = listed ? (const int32_t *)((char *)d_ws + lay.prm + PRM_TILES) : nullptr;
        cudaGraph_t graph = nullptr;
        cudaError_t ce = cudaStreamBeginCapture(di->cap, cudaStreamCaptureModeThreadLocal);
        if (ce != cudaSuccess)
            return cuda_fail(ce, "cudaStreamBeginCapture");
        Timing tm;
        tm.on = (flags & (MANDEL_FLAG_TIMING | MANDEL_FLAG_TIMING_LEAF)) != 0;
        tm.leaf_only = (flags & MANDEL_FLAG_TIMING) == 0;
        int erc = MANDEL_OK;
        if ((flags & (MANDEL_FLAG_TILE_COST | MANDEL_FLAG_TILE_COST_SAMPLED)) && ngroups > 1) {
            // every g*g counter starts at 0 (one group: k_init zeroes them)
            ce = cudaMemsetAsync((char *)d_ws + lay.tile_cost, 0, (size_t)G * 8, di->cap);
            if (ce != cudaSuccess)
                erc = cuda_fail(ce, "cudaMemsetAsync(tile_cost)");
        }
        if (dlist && ngroups > 1 && !erc) { // the device tile list and its length into the parameter block
            char *pb = (char *)d_ws + lay.prm;
            ce = cudaMemcpyAsync(pb + offsetof(DevParams, ntiles), d_ntiles, 4, cudaMemcpyDeviceToDevice, di->cap);
            if (ce == cudaSuccess)
                ce = cudaMemcpyAsync(pb + PRM_TILES, d_tiles_in, (size_t)G * 4, cudaMemcpyDeviceToDevice, di->cap);
            if (ce != cudaSuccess)
                erc = cuda_fail(ce, "cudaMemcpyAsync(device tile list)");
        }
        if (erc) {
        } else if (ngroups == 1) {
            Group grp{lay.hdr, 0, ntiles, d_tiles, cap_tiles};
            erc = enqueue_ask(key, lay, grp, 1, di->sms, di->cap, di->side[0], di->fork[0], &tm);
        } else { // fork one branch per group off the origin stream, join them at the end
            cudaError_t fe = cudaEventRecord(di->start, di->cap);
            size_t unit0 = 0;
            for (int gi = 0; gi < ngroups && !erc && fe == cudaSuccess; ++gi) {
                fe = cudaStreamWaitEvent(di->grp[gi], di->start, 0);
                if (fe != cudaSuccess)
                    break;
                Group grp{lay.hdr + (size_t)gi * 4096, unit0, gcount[(size_t)gi], d_tiles + unit0, gcount[(size_t)gi]};
                erc = enqueue_ask(key, lay, grp, ngroups, di->sms, di->grp[gi], di->side[gi], di->fork[gi], &tm);
                if (!erc)
                    fe = cudaEventRecord(di->join[gi], di->grp[gi]);
                if (!erc && fe == cudaSuccess)
                    fe = cudaStreamWaitEvent(di->cap, di->join[gi], 0);
                unit0 += (size_t)gcount[(size_t)gi];
            }
            if (!erc && fe != cudaSuccess)
                erc = cuda_fail(fe, "group fork/join");
        }
        e.evs = tm.evs;
        e.kinds = tm.kinds;
        e.t_start = tm.start;
        e.t_end = tm.end;
        e.id = ++g_next_id;
        ce = cudaStreamEndCapture(di->cap, &graph);
        if (erc || ce != cudaSuccess) {
            if (graph)
                cudaGraphDestroy(graph);
            free_entry(e);
            return erc ? erc : cuda_fail(ce, "cudaStreamEndCapture");
        }
        ce = cudaGraphInstantiateWithFlags(&e.exec, graph, MANDEL_PRIO ? cudaGraphInstantiateFlagUseNodePriority : 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) {
            free_entry(e);
            return cuda_fail(ce, "cudaGraphInstantiate");
        }
        ++g_captures;
        g_cache.push_back(e);
        hit = &g_cache.back();
    }
    hit->last_use = ++g_clock;
    CK(cudaGraphLaunch(hit->exec, (cudaStream_t)stream));
    if (!hit->evs.empty())
        g_last_timed = hit->id;
    return MANDEL_OK;
}

} // namespace

extern "C" {

int mandel_ask_tiles(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B,
                     const int32_t *h_tile_ids, int32_t n_tiles, int32_t scheme, uint32_t flags, int32_t *d_out,
                     int64_t out_pitch, void *d_ws, size_t ws_bytes, void *stream)
{
    return ask_launch(reg, n, maxdwell, g, r, B, h_tile_ids, n_tiles, nullptr, nullptr, scheme, flags, d_out,
                      out_pitch, d_ws, ws_bytes, stream);
}

int mandel_ask_dtiles(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B,
                      const int32_t *d_tile_ids, const int32_t *d_n_tiles, int32_t scheme, uint32_t flags,
                      int32_t *d_out, int64_t out_pitch, void *d_ws, size_t ws_bytes, void *stream)
{
    if (!d_tile_ids)
        return MANDEL_EINVAL;
    return ask_launch(reg, n, maxdwell, g, r, B, nullptr, 0, d_tile_ids, d_n_tiles, scheme, flags, d_out, out_pitch,
                      d_ws, ws_bytes, stream);
}

int mandel_deal_lpt(const uint64_t *d_costs, int32_t n_tiles, int32_t world, int32_t rank, int32_t *d_tile_ids,
                    int32_t *d_n_tiles, void *stream)
{
    if (!d_costs || !d_tile_ids || !d_n_tiles || n_tiles < 1 || n_tiles > 4096 || world < 1 || world > 64 ||
        rank < 0 || rank >= world)
        return MANDEL_EINVAL;
    k_deal_lpt<<<1, 1024, 0, (cudaStream_t)stream>>>((const unsigned long long *)d_costs, n_tiles, world, rank,
                                                     d_tile_ids, d_n_tiles);
    CK(cudaGetLastError());
    return MANDEL_OK;
}

size_t mandel_ask_tile_costs_offset(int64_t n, int32_t g, int32_t r, int32_t B)
{
    Layout lay;
    if (!make_layout(n, g, r, B, lay))
        return 0;
    return lay.tile_cost;
}

int mandel_ask_kernel_times(float *ms, int32_t *kind_level, int32_t max_kernels)
{
    std::lock_guard<std::mutex> lk(g_mu);
    const Entry *hit = nullptr;
    for (auto &e : g_cache)
        if (e.id == g_last_timed && !e.evs.empty())
            hit = &e;
    if (!hit)
        return -MANDEL_EINVAL;
    for (auto ev : hit->evs)
        CK(cudaEventSynchronize(ev));
    const int nk = (int)hit->kinds.size();
    for (int i = 0; i < nk && i < max_kernels; ++i) {
        float t = 0.0f;
        CK(cudaEventElapsedTime(&t, hit->evs[(size_t)hit->t_start[(size_t)i]],
                                hit->evs[(size_t)hit->t_end[(size_t)i]]));
        if (ms)
            ms[i] = t;
        if (kind_level)
            kind_level[i] = hit->kinds[(size_t)i];
    }
    return nk;
}

int mandel_ask(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B, int32_t *d_out,
               int64_t out_pitch, void *d_ws, size_t ws_bytes, void *stream)
{
    return mandel_ask_tiles(reg, n, maxdwell, g, r, B, nullptr, 0, MANDEL_SCHEME_B200, 0u, d_out, out_pitch, d_ws,
                            ws_bytes, stream);
}

} // extern "C"

namespace {

// u16 host images (mandel_ask_to_host_u16): dst[y][x] = (uint16_t)src[y][x] over the rectangle
// rows [y0, y0+rows) x columns [x0, x0+cols), both buffers addressed with their own pitch
// (elements).  Every dwell is in [1, maxdwell] and maxdwell <= 65535 is checked by the caller,
// so the narrowing is exact.  Four pixels per thread (int4 load, 8-byte store) when the
// rectangle and both pitches are multiples of 4, else one.
__global__ void __launch_bounds__(256) k_to_u16(const int32_t *__restrict__ src, int64_t src_pitch,
                                                uint16_t *__restrict__ dst, int64_t dst_pitch, int64_t y0,
                                                int64_t rows, int64_t x0, int64_t cols, int vec)
{
    const int64_t per_row = vec ? cols / 4 : cols;
    const int64_t total = rows * per_row;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = y0 + t / per_row, c = t % per_row;
        if (vec) {
            const int64_t x = x0 + 4 * c;
            const int4 v = __ldcs(reinterpret_cast<const int4 *>(src + y * src_pitch + x));
            uint2 o;
            o.x = (uint32_t)(v.x & 0xffff) | ((uint32_t)v.y << 16);
            o.y = (uint32_t)(v.z & 0xffff) | ((uint32_t)v.w << 16);
            *reinterpret_cast<uint2 *>(dst + y * dst_pitch + x) = o;
        } else {
            const int64_t x = x0 + c;
            dst[y * dst_pitch + x] = (uint16_t)src[y * src_pitch + x];
        }
    }
}

int to_u16(const int32_t *src, int64_t src_pitch, uint16_t *dst, int64_t dst_pitch, int64_t y0, int64_t rows,
           int64_t x0, int64_t cols, int sms, cudaStream_t s)
{
    const int vec = (x0 % 4 == 0 && cols % 4 == 0 && src_pitch % 4 == 0 && dst_pitch % 4 == 0 &&
                     ((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 7) == 0);
    const int64_t work = rows * (vec ? cols / 4 : cols);
    int64_t grid = (work + 255) / 256;
    const int64_t cap = (int64_t)sms * 8;
    grid = grid < 1 ? 1 : (grid > cap ? cap : grid);
    k_to_u16<<<(unsigned)grid, 256, 0, s>>>(src, src_pitch, dst, dst_pitch, y0, rows, x0, cols, vec);
    CK(cudaGetLastError());
    return MANDEL_OK;
}

// mandel_ask_to_host (T = int32_t: d_stage unused) and mandel_ask_to_host_u16 (T = uint16_t:
// each finished band or tile is narrowed into d_stage, pitch n, on the copy stream, and the
// copy reads d_stage -- half the PCIe bytes).
template <typename T>
int ask_to_host_impl(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B,
                     const int32_t *h_tile_ids, int32_t n_tiles, int32_t scheme, int32_t *d_out, int64_t out_pitch,
                     void *d_ws, size_t ws_bytes, uint16_t *d_stage, T *h_out, void *stream)
{
    constexpr bool U16 = sizeof(T) == 2;
    if (!h_out || (U16 && (!d_stage || maxdwell > 65535)))
        return MANDEL_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t E = sizeof(T);
    if (h_tile_ids) { // only the tiles' pixels: one 2-D copy per tile
        int rc = mandel_ask_tiles(reg, n, maxdwell, g, r, B, h_tile_ids, n_tiles, scheme, 0u, d_out, out_pitch, d_ws,
                                  ws_bytes, stream);
        if (rc)
            return rc;
        int dev = 0, sms = 148;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int64_t d0 = n / g;
        for (int32_t i = 0; i < n_tiles; ++i) {
            const int64_t gy = h_tile_ids[i] / g, gx = h_tile_ids[i] % g;
            const size_t off_h = (size_t)(gy * d0) * (size_t)n + (size_t)(gx * d0);
            const size_t off_d = (size_t)(gy * d0) * (size_t)out_pitch + (size_t)(gx * d0);
            const void *src = d_out + off_d;
            size_t spitch = (size_t)out_pitch * 4;
            if (U16) {
                rc = to_u16(d_out, out_pitch, d_stage, n, gy * d0, d0, gx * d0, d0, sms, st);
                if (rc)
                    return rc;
                src = d_stage + off_h;
                spitch = (size_t)n * 2;
            }
            CK(cudaMemcpy2DAsync(h_out + off_h, (size_t)n * E, src, spitch, (size_t)d0 * E, (size_t)d0,
                                 cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
        return MANDEL_OK;
    }
    // Whole image: bands of level-0 tile rows, each an independent mandel_ask_tiles call
    // (level-0 regions never interact, so the image is the same); the device->host copy of
    // band b runs on a copy stream while band b+1 computes, in chunks of <= 256 MB (the
    // copy, ~55 GB/s over PCIe, dominates this call).
    if (!valid_grb(n, g, r, B) || !valid_region(reg) || !d_out || out_pitch < n)
        return MANDEL_EINVAL;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    DevInfo *di = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int rc = dev_info(dev, di);
        if (rc)
            return rc;
    }
    // bands of level-0 tile rows: only the first band's compute is exposed before the copy
    // stream starts, so more bands hide more of it (MANDEL_E2E_BANDS, a power of two <= 64;
    // C3: 4 bands 80.6 ms, 8 bands 78.0 ms, 16 bands 78.0 ms)
#ifndef MANDEL_E2E_BANDS
#define MANDEL_E2E_BANDS 8
#endif
    const int K = g >= MANDEL_E2E_BANDS ? MANDEL_E2E_BANDS : g, rows_per_band = g / K;
    const int64_t d0 = n / g;
    const int64_t chunk_rows = ((int64_t)1 << 26) / n > 0 ? ((int64_t)1 << 26) / n : 1;
    std::vector<int32_t> tiles;
    NvtxRange nv(U16 ? "mandel_ask_to_host_u16 (bands)" : "mandel_ask_to_host (bands)");
    for (int b = 0; b < K; ++b) {
        tiles.clear();
        for (int gy = b * rows_per_band; gy < (b + 1) * rows_per_band; ++gy)
            for (int gx = 0; gx < g; ++gx)
                tiles.push_back(gy * g + gx);
        int rc = mandel_ask_tiles(reg, n, maxdwell, g, r, B, tiles.data(), (int32_t)tiles.size(), scheme, 0u, d_out,
                                  out_pitch, d_ws, ws_bytes, stream);
        if (rc)
            return rc;
        CK(cudaEventRecord(di->band[b], st));
        CK(cudaStreamWaitEvent(di->copy, di->band[b], 0));
        const int64_t y0 = (int64_t)b * rows_per_band * d0, y1 = (int64_t)(b + 1) * rows_per_band * d0;
        if (U16) {
            rc = to_u16(d_out, out_pitch, d_stage, n, y0, y1 - y0, 0, n, di->sms, di->copy);
            if (rc)
                return rc;
        }
        for (int64_t y = y0; y < y1; y += chunk_rows) {
            const int64_t rows = y + chunk_rows <= y1 ? chunk_rows : y1 - y;
            if (U16)
                CK(cudaMemcpyAsync(h_out + (size_t)y * (size_t)n, d_stage + (size_t)y * (size_t)n,
                                   (size_t)rows * (size_t)n * 2, cudaMemcpyDeviceToHost, di->copy));
            else
                CK(cudaMemcpy2DAsync(h_out + (size_t)y * (size_t)n, (size_t)n * 4,
                                     d_out + (size_t)y * (size_t)out_pitch, (size_t)out_pitch * 4, (size_t)n * 4,
                                     (size_t)rows, cudaMemcpyDeviceToHost, di->copy));
        }
    }
    CK(cudaEventRecord(di->copied, di->copy));
    CK(cudaStreamWaitEvent(st, di->copied, 0));
    CK(cudaStreamSynchronize(st));
    return MANDEL_OK;
}

} // namespace

extern "C" {

int mandel_ask_to_host(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B,
                       const int32_t *h_tile_ids, int32_t n_tiles, int32_t scheme, int32_t *d_out, int64_t out_pitch,
                       void *d_ws, size_t ws_bytes, int32_t *h_out, void *stream)
{
    return ask_to_host_impl<int32_t>(reg, n, maxdwell, g, r, B, h_tile_ids, n_tiles, scheme, d_out, out_pitch, d_ws,
                                     ws_bytes, nullptr, h_out, stream);
}

int mandel_ask_to_host_u16(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B,
                           const int32_t *h_tile_ids, int32_t n_tiles, int32_t scheme, int32_t *d_out,
                           int64_t out_pitch, void *d_ws, size_t ws_bytes, uint16_t *d_stage, uint16_t *h_out,
                           void *stream)
{
    return ask_to_host_impl<uint16_t>(reg, n, maxdwell, g, r, B, h_tile_ids, n_tiles, scheme, d_out, out_pitch, d_ws,
                                      ws_bytes, d_stage, h_out, stream);
}

int mandel_ask_last_stats(const void *d_ws, mandel_level_stats *h_out, int32_t max_levels, void *stream)
{
    if (!d_ws || (!h_out && max_levels > 0) || max_levels < 0)
        return -MANDEL_EINVAL;
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    WsHeader h;
    CK(cudaMemcpy(&h, d_ws, sizeof h, cudaMemcpyDeviceToHost));
    if (h.magic != WS_MAGIC || h.levels < 1 || h.levels > (uint32_t)MAXL || h.ngroups < 1 ||
        h.ngroups > (uint32_t)MAXG)
        return -MANDEL_EINVAL;
    // sum the counters of every group's header (group 0's header carries the group count)
    std::vector<WsHeader> hs(h.ngroups);
    CK(cudaMemcpy2D(hs.data(), sizeof(WsHeader), d_ws, 4096, sizeof(WsHeader), h.ngroups,
                    cudaMemcpyDeviceToHost));
    const int L = (int)h.levels;
    int64_t d = (int64_t)h.n / h.g;
    int64_t regions = 0;
    for (const auto &hg : hs)
        regions += hg.ntiles;
    for (int l = 0; l < L && l < max_levels; ++l) {
        mandel_level_stats &s = h_out[l];
        s.level = l;
        s.side = (int32_t)d;
        s.regions_in = regions;
        s.filled = s.subdivided = s.leaves = s.border_px = s.border_iters = s.leaf_px = s.leaf_iters = 0;
        for (const auto &hg : hs) {
            s.filled += hg.n_fill[l];
            s.subdivided += hg.n_subdiv[l];
            s.leaves += (l == L - 1) ? hg.n_leaf : 0;
            s.border_px += (int64_t)hg.border_px[l];
            s.border_iters += (int64_t)hg.border_iters[l];
            s.leaf_px += (l == L - 1) ? (int64_t)hg.leaf_px : 0;
            s.leaf_iters += (l == L - 1) ? (int64_t)hg.leaf_iters : 0;
        }
        regions = s.subdivided * h.r * h.r;
        d /= h.r;
    }
    return L;
}

int mandel_ask_tile_costs(const void *d_ws, uint64_t *h_costs, int32_t max_tiles, void *stream)
{
    if (!d_ws || !h_costs || max_tiles < 0)
        return -MANDEL_EINVAL;
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    WsHeader h;
    CK(cudaMemcpy(&h, d_ws, sizeof h, cudaMemcpyDeviceToHost));
    if (h.magic != WS_MAGIC)
        return -MANDEL_EINVAL;
    Layout lay;
    if (!make_layout((int64_t)h.n, (int32_t)h.g, (int32_t)h.r, (int32_t)h.B, lay))
        return -MANDEL_EINVAL;
    const int G = (int)(h.g * h.g);
    const int cnt = G < max_tiles ? G : max_tiles;
    CK(cudaMemcpy(h_costs, (const char *)d_ws + lay.tile_cost, (size_t)cnt * 8, cudaMemcpyDeviceToHost));
    return G;
}

const char *mandel_strerror(int code)
{
    switch (code) {
    case MANDEL_OK:
        return "ok";
    case MANDEL_EINVAL:
        return "invalid argument";
    case MANDEL_EWORKSPACE:
        return "workspace too small";
    case MANDEL_ECUDA:
        return "CUDA error";
    default:
        return "unknown error";
    }
}

const char *mandel_last_cuda_error(void) { return g_cuda_err; }

#ifdef MANDEL_RF_TRACE
// Debug builds only (not part of include/mandel.h): copy the refill trace of the last
// traced launch ({start, exhausted, end, pixels | active << 40} per warp) to host memory.
int mandel_debug_rf_trace(unsigned long long *h) // 16 x 8192 x 4 u64
{
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpyFromSymbol(h, g_rf_trace, sizeof(g_rf_trace)));
    return MANDEL_OK;
}
int mandel_debug_rf_trace_clear(void)
{
    static unsigned long long z[16][8192][4];
    CK(cudaMemcpyToSymbol(g_rf_trace, z, sizeof z));
    return MANDEL_OK;
}
#endif

void mandel_shutdown(void)
{
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto &e : g_cache)
        free_entry(e);
    g_cache.clear();
    for (auto &dp : g_dev) {
        DevInfo &d = *dp;
        if (d.cap)
            cudaStreamDestroy(d.cap);
        if (d.start)
            cudaEventDestroy(d.start);
        for (int i = 0; i < MAXG; ++i) {
            if (d.grp[i])
                cudaStreamDestroy(d.grp[i]);
            if (d.side[i])
                cudaStreamDestroy(d.side[i]);
            if (d.fork[i])
                cudaEventDestroy(d.fork[i]);
            if (d.join[i])
                cudaEventDestroy(d.join[i]);
        }
        if (d.copy)
            cudaStreamDestroy(d.copy);
        for (auto ev : d.band)
            if (ev)
                cudaEventDestroy(ev);
        if (d.copied)
            cudaEventDestroy(d.copied);
    }
    g_dev.clear();
}

} // extern "C"
