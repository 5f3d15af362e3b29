// flow.cuh -- MANDEL_SCHEME_FLOW: the B200 scheme's work (border reuse, lane-refill dwell
// engine, warp classification, fills) as ONE persistent dataflow kernel.
//
// The level-synchronous loop waits, at every level, for the level's slowest
// pixel: at one rank's share of a multi-GPU run each of the 7-8 border levels costs
// 0.12-0.17 ms however little work it holds (tools/level_profile.py).  Decisions are
// region-local (a region's fate depends only on its own ring), so nothing requires level
// l+1 of one region to wait for level l of another.  Here a region's next step starts as
// soon as its own ring is complete:
//
//   * work is a stream of UNITS (<= FLOW_U pixels of one task, or one piece of a fill) in a
//     workspace array; producers reserve unit slots with an atomicAdd, write the descriptors
//     and advance a publication watermark in reservation order; persistent warps claim unit
//     indices with an atomicAdd on a cursor and wait until the watermark passes them;
//   * a TASK is the set of pixels one step computes: a level-0 tile's ring (kind 0), the
//     new division lines of a subdivided parent (kind 1, the B200 border reuse of §4.1), or
//     a leaf interior (kind 2); each task counts its pixels down as their dwells are stored
//     (one warp-aggregated atomicSub per task per replay batch);
//   * the warp that completes a task classifies the regions whose rings it completed (the
//     tile, or the r^2 children of the parent) exactly as k_b200_classify does, and
//     publishes their successors: a fill, a kind-1 task, or a kind-2 task;
//   * the kernel ends when no task is pending and every published unit was claimed.
//
// Every pixel's dwell and every region's decision are those of the level-synchronous B200
// scheme, so the image is identical (and the oracle's); only the order of work changes.
#pragma once
#include "ask_kernels.cuh"

namespace mandel {

constexpr uint32_t FLOW_U = 64;        // pixels per unit (= a warp's slots)
constexpr uint32_t FLOW_PIECE = 4096;  // fill elements (int4 or int) per fill unit
constexpr uint32_t FLOW_FILLBIT = 0x80000000u;
constexpr uint32_t FLOW_RINGBIT = 0x80000000u; // parked point: its pixel is a ring pixel
constexpr uint32_t FLOW_NONE = 0xffffffffu;

// Records written during the kernel (tasks, fills, unit descriptors) are always read with
// ld.global.cg (L2): L1 is not coherent, and a line holding several records may have been
// cached before a neighbouring record was written.
struct FlowTask {
    uint32_t origin;    // packed x | y << 16
    uint32_t meta;      // level | kind << 8
    uint32_t npix;
    uint32_t remaining; // pixels whose dwell is not yet stored
};

struct FlowPoint { // a parked chunk-start point (refill.cuh ParkedPoint + its task)
    uint32_t pxy;      // x | y << 16
    float x, y;
    uint32_t it;
    uint32_t task;     // task id | FLOW_RINGBIT
};

__device__ __forceinline__ volatile WsHeader *vhdr(const LevelArgs &a) { return (volatile WsHeader *)a.hdr; }

// GPU-scope ordered atomics / loads (PTX memory model).  A lane's pixel stores are ordered
// before another lane's release by the warp barrier (bar.warp.sync orders memory among the
// participating threads) and release / acquire are cumulative, so ONE ordered operation per
// warp replaces a full fence on every lane.
__device__ __forceinline__ uint32_t atom_sub_release(uint32_t *p, uint32_t v)
{
    uint32_t old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(0u - v) : "memory");
    return old;
}
__device__ __forceinline__ void red_add_release(uint32_t *p, uint32_t v)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Side of the regions of level l.
__device__ __forceinline__ int flow_side(const LevelArgs &a, int l) { return a.d0 >> (l * a.r_log2); }

// ---------------------------------------------------------------------------- publishing
// Warp-cooperative (all 32 lanes, uniform arguments).  Producers reserve unit slots with an
// atomicAdd on f_unit_alloc and write each descriptor with one 16-byte store whose first word
// is FLOW_READY; a consumer that claimed unit u waits for that word, reads the descriptor and
// zeroes it again, so the array is all-zero between calls (k_flow_clear zeroes it whenever
// the workspace is not known to be clean, e.g. on first use).  pending is raised before any
// unit of a task is visible.
constexpr uint32_t FLOW_READY = 0x52454459u;   // "READ"
constexpr uint32_t FLOW_CLEAN = 0x434c454eu;   // unit array all zero (the workspace marker)

__device__ __forceinline__ void flow_publish_units(const LevelArgs &a, uint32_t nu, uint32_t y, uint32_t total,
                                                   uint32_t per)
{
    const int lane = threadIdx.x & 31;
    uint32_t u0 = 0;
    if (lane == 0)
        u0 = atomicAdd(&a.hdr->f_unit_alloc, nu);
    // the task / fill record (written by lane 0) before any descriptor: lane 0 fences, the
    // warp barrier orders the other lanes' descriptor stores after it
    if (lane == 0)
        fence_acq_rel();
    __syncwarp();
    u0 = __shfl_sync(0xffffffffu, u0, 0);
    for (uint32_t i = lane; i < nu; i += 32) {
        const uint32_t st = i * per;
        __stcg(&a.funit[u0 + i], make_uint4(FLOW_READY, y, st, min(per, total - st)));
    }
}

__device__ __forceinline__ void flow_publish_task(const LevelArgs &a, uint32_t origin, int level, int kind,
                                                  uint32_t npix)
{
    const int lane = threadIdx.x & 31;
    uint32_t tid = 0;
    if (lane == 0) {
        atomicAdd(&a.hdr->f_pending, 1u);
        tid = atomicAdd(&a.hdr->f_task_alloc, 1u);
        FlowTask t;
        t.origin = origin;
        t.meta = (uint32_t)level | ((uint32_t)kind << 8);
        t.npix = npix;
        t.remaining = npix;
        a.ftask[tid] = t;
    }
    tid = __shfl_sync(0xffffffffu, tid, 0);
    flow_publish_units(a, (npix + FLOW_U - 1) / FLOW_U, tid, npix, FLOW_U);
}

// Fill of a uniform region (terminal work T) as FLOW_PIECE-element units.
__device__ __forceinline__ void flow_publish_fill(const LevelArgs &a, uint32_t origin, int d, int v)
{
    const int lane = threadIdx.x & 31;
    const bool vec = a.fill_vec && d >= 4;
    const uint32_t elems = vec ? (uint32_t)d * (uint32_t)d / 4u : (uint32_t)d * (uint32_t)d;
    uint32_t fid = 0;
    if (lane == 0) {
        fid = atomicAdd(&a.hdr->f_fill_alloc, 1u);
        a.ffill[fid] = make_uint2(origin, (uint32_t)v);
    }
    fid = __shfl_sync(0xffffffffu, fid, 0);
    int lg = 0;
    while ((1 << lg) < d)
        ++lg;
    flow_publish_units(a, (elems + FLOW_PIECE - 1) / FLOW_PIECE, FLOW_FILLBIT | ((uint32_t)lg << 26) | fid, elems,
                       FLOW_PIECE);
}

// Warp-cooperative fill of one fill unit.
__device__ __forceinline__ void flow_do_fill(const LevelArgs &a, uint4 u)
{
    const int lane = threadIdx.x & 31;
    const uint32_t fid = u.y & ((1u << 26) - 1u);
    const int lg = (int)((u.y >> 26) & 31u), d = 1 << lg;
    const uint2 f = __ldcg(&a.ffill[fid]); // L2: the record may be newer than an L1 line
    const int x0 = unpack_x(f.x), y0 = unpack_y(f.x), v = (int)f.y;
    if (a.fill_vec && d >= 4) {
        const int lq = lg - 2; // int4 per row = d / 4
        const int4 v4 = make_int4(v, v, v, v);
        for (uint32_t i = lane; i < u.w; i += 32) {
            const uint32_t e = u.z + i;
            const int row = (int)(e >> lq), c = (int)(e & ((1u << lq) - 1u));
            __stcs(reinterpret_cast<int4 *>(a.out + (long long)(y0 + row) * a.pitch + x0) + c, v4);
        }
    } else {
        for (uint32_t i = lane; i < u.w; i += 32) {
            const uint32_t e = u.z + i;
            const int row = (int)(e >> lg), c = (int)(e & ((1u << lg) - 1u));
            a.out[(long long)(y0 + row) * a.pitch + x0 + c] = v;
        }
    }
}

// ---------------------------------------------------------------------------- decisions
// Classify one region from its ring in the image / colT (warp-wide min and
// max, as k_b200_classify) and publish what follows.  Counters as the level kernels keep them.
__device__ __forceinline__ void flow_classify(const LevelArgs &a, uint32_t origin, int level)
{
    const int d = flow_side(a, level), ring = 4 * d - 4;
    const int x0 = unpack_x(origin), y0 = unpack_y(origin);
    const int lane = threadIdx.x & 31;
    int lo = INT_MAX, hi = INT_MIN;
    for (int b0 = lane; b0 < ring; b0 += 8 * 32) {
        int v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int b = b0 + j * 32;
            int x, y;
            ring_pixel(b < ring ? b : 0, d, x0, y0, x, y);
            const int *src = (a.colT && b >= 2 * d) ? a.colT + colT_index(a, x, y) : a.out + (long long)y * a.pitch + x;
            v[j] = b < ring ? __ldcg(src) : v[0]; // j = 0 is always in range
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            lo = min(lo, v[j]);
            hi = max(hi, v[j]);
        }
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lo == hi) {
        if (lane == 0)
            atomicAdd(&a.hdr->n_fill[level], 1u);
        flow_publish_fill(a, origin, d, lo);
    } else if (d / a.r >= a.B) {
        if (lane == 0)
            atomicAdd(&a.hdr->n_subdiv[level], 1u);
        flow_publish_task(a, origin, level, 1, new_border_px_per_parent(d, a.r));
    } else {
        if (lane == 0)
            atomicAdd(&a.hdr->n_leaf, 1u);
        if (d > 2)
            flow_publish_task(a, origin, level, 2, (uint32_t)(d - 2) * (uint32_t)(d - 2));
    }
}

// The task tid is complete (every pixel stored and fenced): classify the regions whose rings
// it completed, then retire it.  Warp-cooperative.
__device__ __forceinline__ void flow_complete(const LevelArgs &a, uint32_t tid)
{
    // acquire: the last release on the task's counter (leader's fence, then the warp barrier
    // orders every lane's ring reads after it)
    __syncwarp();
    if ((threadIdx.x & 31) == 0)
        fence_acq_rel(); // acquire: the releases of every pixel of the task
    __syncwarp();
    const uint4 tr = __ldcg(reinterpret_cast<const uint4 *>(&a.ftask[tid])); // L2, never a stale L1 line
    FlowTask t;
    t.origin = tr.x;
    t.meta = tr.y;
    const int level = (int)(t.meta & 255u), kind = (int)(t.meta >> 8);
    if (kind == 0) {
        flow_classify(a, t.origin, 0);
    } else if (kind == 1) { // the r^2 children of a parent of this level
        const int s = flow_side(a, level + 1);
        const int x0 = unpack_x(t.origin), y0 = unpack_y(t.origin);
        for (int c = 0; c < a.r * a.r; ++c)
            flow_classify(a, pack_xy(x0 + (c % a.r) * s, y0 + (c / a.r) * s), level + 1);
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) // after the successors are published (release)
        red_add_release(&a.hdr->f_pending, 0xffffffffu);
}

// Pixel of a task: local index loc -> (x, y).  Per-level divisors in a.ffd[4 l + k]:
// k = 0: D - 2, 1: d - 2, 2: r (d - 2) (kind 1, parent side D = d_l, child side d = d_{l+1});
// k = 3: d_l - 2 (kind 2 leaf rows).
__device__ __forceinline__ void flow_map(const LevelArgs &a, uint32_t origin, uint32_t meta, uint32_t loc, int &x,
                                         int &y)
{
    const int level = (int)(meta & 255u), kind = (int)(meta >> 8);
    const int x0 = unpack_x(origin), y0 = unpack_y(origin);
    if (kind == 0) {
        ring_pixel((int)loc, a.d0, x0, y0, x, y);
    } else if (kind == 1) {
        const FastDiv &fcol = a.ffd[4 * level], &fseg = a.ffd[4 * level + 1], &flen = a.ffd[4 * level + 2];
        const int d = flow_side(a, level + 1); // (fseg.d is clamped to >= 1 when d == 2)
        const uint32_t pv = (uint32_t)(2 * (a.r - 1)) * fcol.d;
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
    } else {
        const FastDiv &fm = a.ffd[4 * level + 3];
        const uint32_t row = fdiv(loc, fm);
        x = x0 + 1 + (int)(loc - row * fm.d);
        y = y0 + 1 + (int)row;
    }
}

// Store one finished pixel (+ stats in STATS builds).
template <bool STATS>
__device__ __forceinline__ void flow_store(const LevelArgs &a, uint32_t pxy, uint32_t task, int v)
{
    const int x = (int)(pxy & 0xffffu), y = (int)(pxy >> 16);
    if (task & FLOW_RINGBIT)
        store_ring(a, x, y, v);
    else
        a.out[(long long)y * a.pitch + x] = v;
    if (STATS) {
        const uint32_t meta = __ldcg(&a.ftask[task & ~FLOW_RINGBIT].meta);
        const int level = (int)(meta & 255u), kind = (int)(meta >> 8);
        if (kind == 2) {
            atomicAdd(&a.hdr->leaf_px, 1ull);
            atomicAdd(&a.hdr->leaf_iters, (unsigned long long)v);
        } else {
            const int bl = kind == 0 ? 0 : level + 1;
            atomicAdd(&a.hdr->border_px[bl], 1ull);
            atomicAdd(&a.hdr->border_iters[bl], (unsigned long long)v);
        }
        add_tile_cost(a, x, y, v);
    }
}

// Count the stored pixels down per task (one atomicSub per distinct task of the warp) and
// complete the tasks that reached zero.  tid = FLOW_NONE: no pixel on this lane.
__device__ __forceinline__ void flow_account(const LevelArgs &a, uint32_t tid)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    __syncwarp(); // every lane's pixel stores before the leaders' release (see above)
    const uint32_t key = tid == FLOW_NONE ? FLOW_NONE : (tid & ~FLOW_RINGBIT);
    const unsigned grp = __match_any_sync(FULL, key);
    bool done = false;
    if (key != FLOW_NONE && lane == __ffs(grp) - 1) {
        const uint32_t c = (uint32_t)__popc(grp);
        // release: the warp's pixel stores before the count (the completing warp acquires)
        done = atom_sub_release(&a.ftask[key].remaining, c) == c;
    }
    unsigned dm = __ballot_sync(FULL, done); // (warp barrier: the acquire orders the classify reads)
    while (dm) {
        const int src = __ffs(dm) - 1;
        dm &= dm - 1;
        flow_complete(a, __shfl_sync(FULL, key, src));
    }
}

// replay_batch2 (refill.cuh) on flow points: exact dwell by bisection, store, account.
// The stored pixels' tasks are returned in (t0, t1) for DEFERRED accounting: the release that
// publishes them is issued a compute chunk later, when the stores have drained and the
// release costs little (an immediate release waits for them: ncu showed it dominating).
template <int K, bool STATS>
__device__ __forceinline__ void flow_replay(const LevelArgs &a, const FlowPoint *q, int cnt, unsigned md,
                                            uint32_t &t0, uint32_t &t1)
{
    const int lane = threadIdx.x & 31;
    const bool v0 = lane < cnt, v1 = lane + 32 < cnt;
    t0 = FLOW_NONE;
    t1 = FLOW_NONE;
    if (v0) {
        FlowPoint p0 = q[lane], p1 = p0;
        if (v1)
            p1 = q[lane + 32];
        const f2_t CR = f2_pack(pix_re(a.map, (int)(p0.pxy & 0xffffu)), pix_re(a.map, (int)(p1.pxy & 0xffffu)));
        const f2_t CI = f2_pack(pix_im(a.map, (int)(p0.pxy >> 16)), pix_im(a.map, (int)(p1.pxy >> 16)));
        f2_t BX = f2_pack(p0.x, p1.x), BY = f2_pack(p0.y, p1.y);
        f2_t BX2 = f2_mul(BX, BX), BY2 = f2_mul(BY, BY);
        unsigned lo0 = p0.it, lo1 = p1.it;
#pragma unroll
        for (int h = K / 2; h >= 1; h /= 2) {
            f2_t X = BX, Y = BY, X2 = BX2, Y2 = BY2;
#pragma unroll
            for (int k = 0; k < h; ++k)
                MANDEL_STEP2(X, Y, X2, Y2, CR, CI);
            float m0, m1;
            f2_unpack(f2_add(X2, Y2), m0, m1);
            const bool hit0 = !(m0 <= 4.0f) || lo0 + (unsigned)h >= md;
            const bool hit1 = !(m1 <= 4.0f) || lo1 + (unsigned)h >= md;
            float a0, a1, b0, b1;
            f2_unpack(X, a0, a1);
            f2_unpack(BX, b0, b1);
            BX = f2_pack(hit0 ? b0 : a0, hit1 ? b1 : a1);
            f2_unpack(Y, a0, a1);
            f2_unpack(BY, b0, b1);
            BY = f2_pack(hit0 ? b0 : a0, hit1 ? b1 : a1);
            f2_unpack(X2, a0, a1);
            f2_unpack(BX2, b0, b1);
            BX2 = f2_pack(hit0 ? b0 : a0, hit1 ? b1 : a1);
            f2_unpack(Y2, a0, a1);
            f2_unpack(BY2, b0, b1);
            BY2 = f2_pack(hit0 ? b0 : a0, hit1 ? b1 : a1);
            lo0 += hit0 ? 0u : (unsigned)h;
            lo1 += hit1 ? 0u : (unsigned)h;
        }
        flow_store<STATS>(a, p0.pxy, p0.task, (int)(lo0 + 1u));
        t0 = p0.task;
        if (v1) {
            flow_store<STATS>(a, p1.pxy, p1.task, (int)(lo1 + 1u));
            t1 = p1.task;
        }
    }
    __syncwarp();
}

// Account the deferred tasks (pa0, pa1) of the last replay, if any.
__device__ __forceinline__ void flow_flush(const LevelArgs &a, uint32_t &pa0, uint32_t &pa1)
{
    if (__any_sync(0xffffffffu, (pa0 & pa1) != FLOW_NONE)) {
        flow_account(a, pa0);
        flow_account(a, pa1);
    }
    pa0 = pa1 = FLOW_NONE;
}

// ---------------------------------------------------------------------------- kernels
// Zero the unit array unless the workspace marker says the previous flow call left it clean.
__global__ void __launch_bounds__(256) k_flow_clear(LevelArgs a, size_t nunits)
{
    if (*((volatile uint32_t *)a.fmark) == FLOW_CLEAN)
        return;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nunits; i += (size_t)gridDim.x * blockDim.x)
        a.funit[i] = make_uint4(0u, 0u, 0u, 0u);
}

// Publish the level-0 tasks (the rings of the call's tiles, olt_in from k_init) and the
// per-level divisors.  One warp per tile.
__global__ void __launch_bounds__(256) k_flow_init(LevelArgs a)
{
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w == 0 && lane < a.levels) {
        const int l = lane, D = flow_side(a, l), d = D / a.r;
        a.ffd[4 * l] = make_fastdiv((uint32_t)max(D - 2, 1));
        a.ffd[4 * l + 1] = make_fastdiv((uint32_t)max(d - 2, 1));
        a.ffd[4 * l + 2] = make_fastdiv((uint32_t)max(a.r * (d - 2), 1));
        a.ffd[4 * l + 3] = make_fastdiv((uint32_t)max(D - 2, 1));
    }
    if (w == 0 && lane == 0)
        *a.fmark = 0u; // dirty until k_flow's last warp has exited
    if (w < a.ntiles)
        flow_publish_task(a, a.olt_in[w], 0, 0, (uint32_t)(4 * a.d0 - 4));
}

// The persistent dataflow kernel: refill_loop2 (refill.cuh) whose work source is the unit
// stream, with completion accounting and classification in place of the level barrier.
#ifndef MANDEL_FLOW_MINB
#define MANDEL_FLOW_MINB 2
#endif
template <bool STATS>
__global__ void __launch_bounds__(RF_TPB, MANDEL_FLOW_MINB) k_flow(LevelArgs a)
{
    constexpr int K = MANDEL_RFL_K, T = MANDEL_RFL2_T;
    __shared__ FlowPoint s_q[RF_TPB / 32][RF2_QCAP];
    FlowPoint *q = s_q[threadIdx.x >> 5];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned md = (unsigned)a.maxdwell;
    volatile WsHeader *vh = vhdr(a);

    // current unit window (warp-uniform): pixels [pos, end) of task utask
    uint32_t pos = 0, end = 0, utask = 0, uorigin = 0, umeta = 0;
    uint32_t claim = FLOW_NONE; // claimed unit index not yet published
    bool finished = false;      // nothing pending anywhere and every unit claimed
    int qn = 0;
    uint32_t pa0 = FLOW_NONE, pa1 = FLOW_NONE; // deferred accounting (flow_replay)

    bool has0 = false, has1 = false, fin0 = false, fin1 = false;
    uint32_t pxy0 = 0, pxy1 = 0, tk0 = 0, tk1 = 0;
    unsigned it0 = 0, it1 = 0, sit0 = 0, sit1 = 0;
    float sx0 = 0.f, sy0 = 0.f, sx1 = 0.f, sy1 = 0.f;
    f2_t X = 0, Y = 0, X2 = 0, Y2 = 0, CR = 0, CI = 0;

    while (true) {
        // ---------------------------------------------------------------- park
        flow_flush(a, pa0, pa1); // the previous round's replay (its stores have drained)
        const unsigned f0 = __ballot_sync(FULL, fin0), f1 = __ballot_sync(FULL, fin1);
        if (f0 | f1) {
            const int n0 = __popc(f0);
            if (fin0) {
                FlowPoint &e = q[qn + __popc(f0 & lt)];
                e.pxy = pxy0;
                e.x = sx0;
                e.y = sy0;
                e.it = sit0;
                e.task = tk0;
                has0 = false;
                fin0 = false;
            }
            if (fin1) {
                FlowPoint &e = q[qn + n0 + __popc(f1 & lt)];
                e.pxy = pxy1;
                e.x = sx1;
                e.y = sy1;
                e.it = sit1;
                e.task = tk1;
                has1 = false;
                fin1 = false;
            }
            qn += n0 + __popc(f1);
            __syncwarp();
            if (qn >= 64) {
                qn -= 64;
                flow_replay<K, STATS>(a, q + qn, 64, md, pa0, pa1);
            }
        }
        // ---------------------------------------------------------------- refill
        bool starved = false;
        unsigned need0 = __ballot_sync(FULL, !has0), need1 = __ballot_sync(FULL, !has1);
        while ((need0 | need1) && !finished) {
            if (pos >= end) {
                // claim the next unit (once) and wait for it to be published
                uint4 u = make_uint4(0, 0, 0, 0);
                if (lane == 0) {
                    if (claim == FLOW_NONE)
                        claim = atomicAdd(&a.hdr->f_cursor, 1u);
                    // (the task record read below is address-dependent on this load, and the
                    // producer fenced it before the descriptor)
                    u = __ldcg(&a.funit[claim]);
                    if (u.x == FLOW_READY) {
                        __stcg(&a.funit[claim], make_uint4(0u, 0u, 0u, 0u));
                    } else { // not published yet -- or never: nothing pending anywhere
                        const uint32_t pend = ld_acquire(&a.hdr->f_pending);
                        u.x = (pend == 0 && claim >= vh->f_unit_alloc) ? 1u : 0u;
                        u.y = FLOW_NONE;
                    }
                }
                u.x = __shfl_sync(FULL, u.x, 0);
                u.y = __shfl_sync(FULL, u.y, 0);
                u.z = __shfl_sync(FULL, u.z, 0);
                u.w = __shfl_sync(FULL, u.w, 0);
                if (u.y == FLOW_NONE) {
                    if (u.x == 1u)
                        finished = true;
                    else
                        starved = true;
                    break;
                }
                claim = FLOW_NONE;
                if (u.y & FLOW_FILLBIT) {
                    flow_do_fill(a, u);
                    continue;
                }
                utask = u.y;
                const uint2 t = __ldcg(reinterpret_cast<const uint2 *>(&a.ftask[utask]));
                uorigin = t.x;
                umeta = t.y;
                pos = u.z;
                end = u.z + u.w;
            }
            const unsigned c0 = __popc(need0);
            const unsigned cnt = c0 + __popc(need1);
            const unsigned avail = end - pos;
            const unsigned take = avail < cnt ? avail : cnt;
            const unsigned r0 = __popc(need0 & lt), r1 = c0 + __popc(need1 & lt);
            const uint32_t tkv = utask | ((umeta >> 8) != 2u ? FLOW_RINGBIT : 0u);
            float cr0, ci0, cr1, ci1;
            f2_unpack(CR, cr0, cr1);
            f2_unpack(CI, ci0, ci1);
            bool new0 = false, new1 = false;
            uint32_t done0 = FLOW_NONE, done1 = FLOW_NONE;
#define FLOW_FETCH(SLOT, RK)                                                                   \
    if (!has##SLOT && RK < take) {                                                             \
        int px, py;                                                                            \
        flow_map(a, uorigin, umeta, pos + RK, px, py);                                         \
        const float cr = pix_re(a.map, px), ci = pix_im(a.map, py);                            \
        pxy##SLOT = (uint32_t)px | ((uint32_t)py << 16);                                       \
        tk##SLOT = tkv;                                                                        \
        if (__fadd_rn(__fmul_rn(cr, cr), __fmul_rn(ci, ci)) <= 3.9f) {                         \
            has##SLOT = new##SLOT = true;                                                      \
            cr##SLOT = cr;                                                                     \
            ci##SLOT = ci;                                                                     \
        } else { /* per-step loop (escape permanence not guaranteed) */                        \
            flow_store<STATS>(a, pxy##SLOT, tkv, dwell_per_step<K>(cr, ci, a.maxdwell));       \
            done##SLOT = tkv;                                                                  \
        }                                                                                      \
    }
            FLOW_FETCH(0, r0)
            FLOW_FETCH(1, r1)
            if (__any_sync(FULL, (done0 & done1) != FLOW_NONE)) { // rare: |c|^2 > 3.9 pixels
                flow_account(a, done0);
                flow_account(a, done1);
            }
#undef FLOW_FETCH
            if (__any_sync(FULL, new0 | new1)) {
                CR = f2_pack(cr0, cr1);
                CI = f2_pack(ci0, ci1);
                float a0, a1;
#define RF2_ZERO(V)                                                                            \
    f2_unpack(V, a0, a1);                                                                      \
    V = f2_pack(new0 ? 0.0f : a0, new1 ? 0.0f : a1);
                RF2_ZERO(X)
                RF2_ZERO(Y)
                RF2_ZERO(X2)
                RF2_ZERO(Y2)
#undef RF2_ZERO
                it0 = new0 ? 0u : it0;
                it1 = new1 ? 0u : it1;
            }
            pos += take;
            need0 = __ballot_sync(FULL, !has0);
            need1 = __ballot_sync(FULL, !has1);
        }
        const unsigned a0m = __ballot_sync(FULL, has0), a1m = __ballot_sync(FULL, has1);
        // no new work right now: replay what is queued, its tasks may be the ones others wait for
        if ((starved || finished) && qn > 0) {
            while (qn > 0) { // (accounted at once: other warps wait for these tasks)
                flow_flush(a, pa0, pa1); // (the park phase's replay, if any)
                const int c = qn < 64 ? qn : 64;
                qn -= c;
                flow_replay<K, STATS>(a, q + qn, c, md, pa0, pa1);
                flow_flush(a, pa0, pa1);
            }
        }
        if (!(a0m | a1m)) {
            if (finished)
                break;
            __nanosleep(200);
            continue;
        }
        // ---------------------------------------------------------------- compute
        const int thresh = (starved || finished) ? 1 : T;
        const bool live0 = has0, live1 = has1;
        while (true) {
            float xl, xh, yl, yh;
            f2_unpack(X, xl, xh);
            f2_unpack(Y, yl, yh);
            const bool keep0 = fin0 || !live0, keep1 = fin1 || !live1;
            sx0 = keep0 ? sx0 : xl;
            sy0 = keep0 ? sy0 : yl;
            sit0 = keep0 ? sit0 : it0;
            sx1 = keep1 ? sx1 : xh;
            sy1 = keep1 ? sy1 : yh;
            sit1 = keep1 ? sit1 : it1;
#pragma unroll
            for (int k = 0; k < K; ++k)
                MANDEL_STEP2(X, Y, X2, Y2, CR, CI);
            it0 += K;
            it1 += K;
            float m0, m1;
            f2_unpack(f2_add(X2, Y2), m0, m1);
            fin0 = live0 && (fin0 || !(m0 <= 4.0f) || it0 >= md);
            fin1 = live1 && (fin1 || !(m1 <= 4.0f) || it1 >= md);
            const unsigned g0 = __ballot_sync(FULL, fin0), g1 = __ballot_sync(FULL, fin1);
            if ((g0 == a0m && g1 == a1m) || __popc(g0) + __popc(g1) >= thresh)
                break;
        }
    }
    // every descriptor this call published was read and zeroed: mark the array clean
    if (lane == 0) {
        __threadfence();
        if (atomicAdd(&a.hdr->f_exited, 1u) == (gridDim.x * blockDim.x >> 5) - 1u) {
            __threadfence();
            *a.fmark = FLOW_CLEAN;
        }
    }
}

} // namespace mandel
