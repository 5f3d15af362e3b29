// refill.cuh -- lane-refill dwell engine for the flat B200 kernels.
//
// The pixels a B200 border or leaf kernel computes are a flat index space [0, total) that a
// Map functor turns into image coordinates.  A plain one-thread-per-pixel kernel loses most
// of the FP32 issue slots to divergence: in a warp, dwells range from 1 to maxdwell exactly
// where ASK leaves and borders are (the fractal boundary: median dwell ~10, 10-20% of the
// pixels at maxdwell), and the warp runs as long as its slowest lane.  Here every warp is
// persistent and keeps its 32 lanes busy:
//
//   * a warp grabs up to CH consecutive indices at a time from a per-launch cursor in the
//     workspace header (one atomicAdd by lane 0) and deals them to its idle lanes in order
//     (ballot + popc rank), so neighbouring pixels run side by side;
//   * busy lanes iterate in unrolled chunks of K steps (dwell.cuh's 7-op step) with one
//     escape test per chunk, keeping the chunk-start point (x, y, iteration);
//   * a lane whose pixel escaped (or reached maxdwell) during the chunk parks that
//     chunk-start point in a per-warp queue in shared memory and is refilled at once, as
//     soon as T lanes are parked;
//   * whenever 32 points are queued the warp replays them together, one lane each: a
//     bisection over the K steps after the chunk start finds the exact first-escape index
//     (escape is permanent), then the dwell is stored.  Replays thus run
//     with all 32 lanes busy instead of stalling the warp once per escaping lane.
//
// The image equals the plain kernels' (each pixel's dwell is a pure function); only which
// lane computes which pixel, and when, changes.  Pixels with |c|^2 > 3.9 (outside every
// config region) bypass the chunked loop and run the per-step loop at fetch time.
#pragma once
#include "dwell.cuh"

namespace mandel {

// Unsigned 32-bit division by a runtime-invariant divisor with a multiply-high
// (Granlund-Montgomery; exact for every n < 2^32, d >= 1).  Host computes the magic.
struct FastDiv {
    uint32_t d, m, s1, s2;
};
__host__ __device__ inline FastDiv make_fastdiv(uint32_t d)
{
    uint32_t l = 0;
    while (l < 32 && (1ull << l) < d)
        ++l;
    FastDiv f;
    f.d = d;
    f.m = (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1ull);
    f.s1 = l < 1 ? l : 1;
    f.s2 = l > 1 ? l - 1 : 0;
    return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f)
{
    const uint32_t t = __umulhi(n, f.m);
    return (t + ((n - t) >> f.s1)) >> f.s2;
}

template <int K>
__device__ __forceinline__ int dwell_per_step(float cr, float ci, int maxdwell)
{
    float x = 0.0f, y = 0.0f, x2 = 0.0f, y2 = 0.0f;
    int i = 0;
    while (i < maxdwell) {
        MANDEL_STEP(x, y, x2, y2, cr, ci);
        ++i;
        if (__fadd_rn(x2, y2) > 4.0f)
            return i;
    }
    return maxdwell;
}

// Late programmatic launch (MANDEL_PDL_LATE, calls with a device tile list): a refill kernel
// waits for its predecessor at entry but lets its successor launch only once its warps find
// the cursor exhausted, i.e. in the level's tail.  Triggered at entry (pdl_entry), the
// successor's blocks are scheduled at once and wait in SM slots for the whole kernel, where
// the overlapped fill kernels would run -- and a device-list call sizes its grids for all g^2
// tiles, so many of them.  (Full images: the early trigger is 1% faster, the late one hides
// less launch latency; profiles/r02_ab_pdl_late.jsonl.)
#ifndef MANDEL_PDL // programmatic dependent launch of the level chain (ask_kernels.cuh)
#define MANDEL_PDL 1
#endif
#ifndef MANDEL_PDL_LATE
#define MANDEL_PDL_LATE 1
#endif
__device__ __forceinline__ void pdl_trigger(bool late)
{
#if MANDEL_PDL && MANDEL_PDL_LATE
    if (late)
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// A parked chunk-start point awaiting its exact replay.
struct ParkedPoint {
    int px, py;
    float x, y;
    unsigned it;
};

constexpr int RF_QCAP = 64; // per-warp queue entries (< 32 left over + < 32 new)

// Scalar engine launch shape (knobs for tools/tune_refill.py): a launch activates
// ~total / (32 PPL) warps, at least MINW per SM (MINW / 4 per sub-partition).
#ifndef MANDEL_RF_PPL
#define MANDEL_RF_PPL 8u
#endif
#ifndef MANDEL_RF_MINW
#define MANDEL_RF_MINW 8u
#endif
#ifndef MANDEL_RF_EXACT
#define MANDEL_RF_EXACT 1
#endif
// Scalar engine: CKPT sub-chunks per K-step chunk.  The orbit is kept at every sub-chunk
// boundary, so a parked point's first escape is located to one sub-chunk from the saved
// points' |z|^2 and the replay bisects K/CKPT steps instead of K (1: plain chunks).
#ifndef MANDEL_RF_DIRECT
#define MANDEL_RF_DIRECT 0 // store unescaped maxdwell points at parking time (measured slower)
#endif
#ifndef MANDEL_RF2_CKPT
#define MANDEL_RF2_CKPT 2 // the same for the packed engine
#endif
#ifndef MANDEL_RF_CKPT
#define MANDEL_RF_CKPT 2
#endif
#ifndef MANDEL_RF_EXACT_PPW
#define MANDEL_RF_EXACT_PPW 1024u // scalar engine: exact grabs below this many pixels per warp
#endif

// SM count of the device the kernels run on (set by the host before capture).
__constant__ int c_num_sms;

#ifdef MANDEL_RF_TRACE
// Debug build only (tools/trace_refill.py): per active warp of the last traced launch,
// {start, cursor exhausted, end} in globaltimer ns and the pixels it computed.
__device__ unsigned long long g_rf_trace[16][8192][4]; // [launch slot][warp rank]
__device__ __forceinline__ unsigned long long rf_now()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// Replay the queued points q[0..cnt) (cnt <= 32), one per lane, and store their dwells.
// A parked point escaped (or reached maxdwell) within the K steps after its chunk start, so
// its dwell is sit + j* with j* the first j in [1, K] where P(j) = "escaped at step j, or
// sit + j >= maxdwell" holds.  P is monotone (escape is permanent), so j* is
// found by bisection: K/2 + K/4 + ... + 1 = K - 1 steps and log2 K tests, instead of up to K
// steps with a test each.  Every lane runs the same instruction sequence (no divergence).
template <int K, class Sink>
__device__ __forceinline__ void replay_batch(const ParkedPoint *q, int cnt, const PixMap &pm, unsigned md,
                                             Sink &sink)
{
    static_assert((K & (K - 1)) == 0, "K must be a power of two");
    const int lane = threadIdx.x & 31;
    if (lane < cnt) {
        const ParkedPoint p = q[lane];
        const float cr = pix_re(pm, p.px), ci = pix_im(pm, p.py);
        float bx = p.x, by = p.y;
        float bx2 = __fmul_rn(bx, bx), by2 = __fmul_rn(by, by); // as the chunk start had them
        unsigned lo = p.it;                                     // P false at lo (not escaped)
#pragma unroll
        for (int h = K / 2; h >= 1; h /= 2) {
            float x = bx, y = by, x2 = bx2, y2 = by2;
#pragma unroll
            for (int k = 0; k < h; ++k)
                MANDEL_STEP(x, y, x2, y2, cr, ci);
            const bool hit = !(__fadd_rn(x2, y2) <= 4.0f) || lo + (unsigned)h >= md;
            if (!hit) { // first hit lies beyond lo + h
                bx = x;
                by = y;
                bx2 = x2;
                by2 = y2;
                lo += (unsigned)h;
            }
        }
        sink(p.px, p.py, (int)(lo + 1u));
    }
    __syncwarp();
}

#ifndef MANDEL_PRE_WINDOW
#define MANDEL_PRE_WINDOW 0xffffffffu // prepass pixels per decision window (default: always on)
#endif
#ifndef MANDEL_PRE_SLOTS
#define MANDEL_PRE_SLOTS 0 // prepass raw pixels per free slot (0: a whole grab)
#endif
#ifndef MANDEL_PRE_COUNT
#define MANDEL_PRE_COUNT 2 // prepass escape test: 0 latch the first escape, 1 integer count, 2 float count
#endif
#ifndef MANDEL_PRE_MINFRAC
#define MANDEL_PRE_MINFRAC 25u // keep the prepass while >= this % of its pixels escape in it
#endif
// A prepass survivor: pixel and its orbit after S steps (x2, y2 are x*x, y*y again).
#ifndef MANDEL_SV_C
#define MANDEL_SV_C 1 // prepass survivors keep c, so dealing them does not recompute it
#endif
struct SvPoint {
    uint32_t pxy; // x | y << 16
    float x, y;
#if MANDEL_SV_C
    float cr, ci; // 20 bytes: the leaf kernel's static shared memory stays below 48 KB
#else
    uint32_t pad;
#endif
};

// Short-pixel prepass (PRE = S > 0): every grab of raw indices is first run
// warp-synchronously, one pixel per lane, for S steps with an escape test after EVERY step
// (exact dwell, no replay); pixels that escape -- 70% of the C3 leaf pixels have dwell <= 16
// -- are stored at once and never enter the refill machinery (fetch, parking, bisection
// replay: ~20 dispatch cycles per pixel); the survivors go to a per-warp buffer sv (CH
// entries) and are dealt to slots with their orbit state at iteration S.  The test
// `!(x2+y2 <= 4)` after step k first fires at the pixel's dwell (escape happens before any
// overflow), so the stored dwell is the per-step definition's.  A warp stops using the
// prepass once fewer than a quarter of its first >= 512 prepass pixels escaped in it
// (boundary-heavy windows such as C5, median leaf dwell 146).
template <int S, class Map, class Sink>
__device__ __forceinline__ int rf2_prepass(uint32_t b, uint32_t e, const PixMap &pm, int maxdwell, const Map &map,
                                           Sink &sink, SvPoint *sv, int &n_esc)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int m = 0, esc = 0;
    for (uint32_t r0 = b; r0 < e; r0 += 32) {
        const uint32_t t = r0 + (uint32_t)lane;
        bool surv = false;
        uint32_t pxy = 0;
        float x = 0.f, y = 0.f;
#if MANDEL_SV_C
        float svcr = 0.f, svci = 0.f;
#endif
        if (t < e) {
            int px, py;
            map(t, px, py);
            pxy = (uint32_t)px | ((uint32_t)py << 16);
            const float cr = pix_re(pm, px), ci = pix_im(pm, py);
            if (__fadd_rn(__fmul_rn(cr, cr), __fmul_rn(ci, ci)) <= 3.9f) {
                float x2 = 0.f, y2 = 0.f;
#if MANDEL_PRE_COUNT == 1
                // escape is permanent (|c|^2 <= 3.9): the steps still inside
                // are exactly the steps before the dwell, so dwell = (their count) + 1
                int in = 0;
#pragma unroll
                for (int k = 1; k <= S; ++k) {
                    MANDEL_STEP(x, y, x2, y2, cr, ci);
                    in += __fadd_rn(x2, y2) <= 4.0f ? 1 : 0;
                }
                const int dw = in < S ? in + 1 : 0;
#elif MANDEL_PRE_COUNT == 2
                // the same count kept in a float (1.0 / 0.0 per step: exact for S < 2^24)
                float inf_ = 0.0f;
#pragma unroll
                for (int k = 1; k <= S; ++k) {
                    MANDEL_STEP(x, y, x2, y2, cr, ci);
                    inf_ = __fadd_rn(inf_, __fadd_rn(x2, y2) <= 4.0f ? 1.0f : 0.0f);
                }
                const int in = (int)inf_;
                const int dw = in < S ? in + 1 : 0;
#else
                int dw = 0;
#pragma unroll
                for (int k = 1; k <= S; ++k) {
                    MANDEL_STEP(x, y, x2, y2, cr, ci);
                    dw = (dw == 0 && !(__fadd_rn(x2, y2) <= 4.0f)) ? k : dw;
                }
#endif
                if (dw) {
                    sink(px, py, dw);
                    ++esc;
                } else {
                    surv = true;
#if MANDEL_SV_C
                    svcr = cr;
                    svci = ci;
#endif
                }
            } else { // per-step loop (escape permanence not guaranteed)
                sink(px, py, dwell_per_step<S>(cr, ci, maxdwell));
                ++esc;
            }
        }
        const unsigned sm = __ballot_sync(FULL, surv);
        if (surv) {
            SvPoint &o = sv[m + __popc(sm & lt)];
            o.pxy = pxy;
            o.x = x;
            o.y = y;
#if MANDEL_SV_C
            o.cr = svcr;
            o.ci = svci;
#endif
        }
        m += __popc(sm);
    }
    n_esc += __reduce_add_sync(FULL, (unsigned)esc);
    __syncwarp();
    return m;
}

// The replay window of a parked point (CKP sub-chunks of KS steps, chunk start (sx, sy, sit),
// kept points ck[c] after (c+1)*KS steps): the sub-chunk after the last kept point not yet
// past the first escape or maxdwell -- P(j) = "escaped by j || sit + j >= md" is monotone.
template <int CKP, int KS>
__device__ __forceinline__ void replay_window(float sx, float sy, unsigned sit, const float *ckx, const float *cky,
                                              unsigned md, float &bx, float &by, unsigned &bit)
{
    bx = sx;
    by = sy;
    bit = sit;
#pragma unroll
    for (int c = 0; c < CKP - 1; ++c) {
        const unsigned jc = sit + (unsigned)((c + 1) * KS);
        const float m = __fadd_rn(__fmul_rn(ckx[c], ckx[c]), __fmul_rn(cky[c], cky[c]));
        if (bit + (unsigned)KS == jc && m <= 4.0f && jc < md) {
            bx = ckx[c];
            by = cky[c];
            bit = jc;
        }
    }
}

// Second prepass stage (MANDEL_PRE2 = S2 > 0): the survivors of rf2_prepass<S1> (orbit at
// iteration S1 in sv[0, m)) run S2 more steps, one per lane, 32 at a time, with the same
// counted escape test; the ones that escape are stored (dwell S1 + count + 1) and the rest are
// compacted in place (orbit at iteration S1 + S2).  Returns the new survivor count.
#ifndef MANDEL_PRE2
#define MANDEL_PRE2 16
#endif
template <int S1, int S2, class Sink>
__device__ __forceinline__ int rf2_prepass_more(SvPoint *sv, int m, const PixMap &pm, Sink &sink, int &n_esc)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int m2 = 0, esc = 0;
    for (int r0 = 0; r0 < m; r0 += 32) {
        const bool valid = r0 + lane < m;
        SvPoint p;
        p.pxy = 0u;
        p.x = p.y = 0.0f;
        if (valid)
            p = sv[r0 + lane];
        bool surv = false;
        if (valid) {
#if MANDEL_SV_C
            const float cr = p.cr, ci = p.ci;
#else
            const float cr = pix_re(pm, (int)(p.pxy & 0xffffu)), ci = pix_im(pm, (int)(p.pxy >> 16));
#endif
            float x = p.x, y = p.y, x2 = __fmul_rn(x, x), y2 = __fmul_rn(y, y);
            float inf_ = 0.0f;
#pragma unroll
            for (int k = 1; k <= S2; ++k) {
                MANDEL_STEP(x, y, x2, y2, cr, ci);
                inf_ = __fadd_rn(inf_, __fadd_rn(x2, y2) <= 4.0f ? 1.0f : 0.0f);
            }
            const int in = (int)inf_;
            if (in < S2) {
                sink((int)(p.pxy & 0xffffu), (int)(p.pxy >> 16), S1 + in + 1);
                ++esc;
            } else {
                surv = true;
                p.x = x;
                p.y = y;
            }
        }
        const unsigned sm = __ballot_sync(FULL, surv); // every lane has read its entry
        if (surv)
            sv[m2 + __popc(sm & lt)] = p;
        m2 += __popc(sm);
    }
    n_esc += __reduce_add_sync(FULL, (unsigned)esc);
    __syncwarp();
    return m2;
}

// Map: __device__ void operator()(uint32_t t, int &x, int &y) const      (t < 2^32)
// Sink: __device__ void operator()(int x, int y, int v)                   (store + stats)
// q: this warp's RF_QCAP-entry queue in shared memory.
// The grab size adapts to the launch: at most CH, but small enough that every warp of the
// grid gets about 4 grabs (small levels -- e.g. one rank's share of a multi-GPU run -- would
// otherwise leave most warps idle while a few run whole grabs of maxdwell pixels), and >= 8.
// PRE > 0: the short-pixel prepass of rf2_prepass on every grab, with
// the per-warp survivor buffer sv (CH entries); survivors are dealt to lanes at iteration PRE.
template <int K, int T, int CH, class Map, class Sink, int PRE = 0>
__device__ __forceinline__ void refill_loop(const PixMap &pm, int maxdwell, uint32_t total,
                                            unsigned long long *cursor, const Map &map, Sink &sink,
                                            ParkedPoint *q, int tslot = 0, SvPoint *sv = nullptr,
                                            bool pdl_late = false, uint32_t ch_cap = 0)
{
    // Active warps: a launch with few pixels per lane runs like a thread-per-pixel kernel
    // (every warp waits for its slowest lane and there is nothing to refill from), so only
    // ~total/(32*PPL) warps work -- but never fewer than 2 per SM sub-partition (592 on
    // B200), below which one warp per scheduler is latency-bound.  Warp w of block b has
    // rank w*gridDim+b, so the active warps spread over all SMs.  (Idle warps return here and
    // still reach the caller's block-wide reductions.)
    constexpr uint32_t PPL = MANDEL_RF_PPL;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t min_active = MANDEL_RF_MINW * (uint32_t)c_num_sms;
    uint32_t active = total / (32u * PPL);
    active = active < min_active ? min_active : active;
    active = active > nwarps ? nwarps : active;
    const uint32_t wrank = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    if (wrank >= active)
        return;
#ifdef MANDEL_RF_TRACE
    unsigned long long tr_start = rf_now(), tr_ex = 0, tr_px = 0;
#endif
    uint32_t grab = total / (4u * active);
    const uint32_t chx = (ch_cap && ch_cap < (uint32_t)CH) ? ch_cap : (uint32_t)CH; // runtime cap <= CH
    grab = grab < 8u ? 8u : (grab > chx ? chx : grab);
    // exact grabs (below) only for launches with few pixels per warp: there a window of long
    // pixels held by one warp is the level's tail; in big launches the extra cursor atomics
    // cost more than the windows (C3's deep border levels)
    const bool exact = MANDEL_RF_EXACT && total / active < MANDEL_RF_EXACT_PPW;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned md = (unsigned)maxdwell;

    uint32_t pos = 0, end = 0; // warp-uniform chunk window [pos, end)
    bool exhausted = false;    // warp-uniform: the cursor ran past total
    int qn = 0;                // warp-uniform queue fill
    const bool use_pre = PRE > 0 && sv != nullptr && maxdwell > PRE;
    uint32_t sv_pos = 0, sv_end = 0; // warp-uniform survivor buffer window
    int pre_esc = 0;

    constexpr int CKP = MANDEL_RF_CKPT, KS = K / CKP; // sub-chunks and their length
    static_assert(CKP >= 1 && K % CKP == 0 && (KS & (KS - 1)) == 0, "CKPT must split K into powers of two");
    bool has = false, fin = false, endok = false;
    int px = 0, py = 0;
    float cr = 0.f, ci = 0.f, x = 0.f, y = 0.f, x2 = 0.f, y2 = 0.f, sx = 0.f, sy = 0.f;
    float ckx[CKP > 1 ? CKP - 1 : 1], cky[CKP > 1 ? CKP - 1 : 1];
#pragma unroll
    for (int c = 0; c < (CKP > 1 ? CKP - 1 : 1); ++c)
        ckx[c] = cky[c] = 0.f;
    unsigned it = 0, sit = 0;

    while (true) {
        // ---------------------------------------------------------------- park + refill
        const unsigned f = __ballot_sync(FULL, fin);
        if (f) {
            // MANDEL_RF_DIRECT: a lane that reached maxdwell unescaped (|z|^2 <= 4 at the
            // chunk end, escape is permanent) has dwell maxdwell: stored at once, no replay
            const bool direct = MANDEL_RF_DIRECT && fin && endok;
            if (direct)
                sink(px, py, (int)md);
            const bool enq = fin && !direct;
            const unsigned fq = MANDEL_RF_DIRECT ? __ballot_sync(FULL, enq) : f;
            if (enq) {
                float bx, by;
                unsigned bit;
                replay_window<CKP, KS>(sx, sy, sit, ckx, cky, md, bx, by, bit);
                ParkedPoint &e = q[qn + __popc(fq & lt)];
                e.px = px;
                e.py = py;
                e.x = bx;
                e.y = by;
                e.it = bit;
            }
            if (fin) {
                has = false;
                fin = false;
            }
            qn += __popc(fq);
            __syncwarp();
            if (qn >= 32) {
                qn -= 32;
                replay_batch<KS>(q + qn, 32, pm, md, sink);
            }
        }
        unsigned need = __ballot_sync(FULL, !has);
        while (need && !exhausted) {
            if constexpr (PRE > 0) {
              if (use_pre) {
                if (sv_pos >= sv_end) { // prepass a fresh grab; its survivors refill the buffer
                    unsigned long long b = 0;
                    if (lane == 0)
                        b = atomicAdd(cursor, (unsigned long long)grab);
                    b = __shfl_sync(FULL, b, 0);
                    if (b >= total) {
                        exhausted = true;
                        pdl_trigger(pdl_late);
                        break;
                    }
                    const uint32_t e = (uint32_t)min(b + (unsigned long long)grab, (unsigned long long)total);
                    sv_pos = 0;
                    sv_end = (uint32_t)rf2_prepass<PRE>((uint32_t)b, e, pm, maxdwell, map, sink, sv, pre_esc);
                    continue;
                }
                // deal survivors (orbit at iteration PRE) to idle lanes
                const unsigned cnt = __popc(need);
                const unsigned avail = sv_end - sv_pos;
                const unsigned take = avail < cnt ? avail : cnt;
                const unsigned rank = __popc(need & lt);
                if (!has && rank < take) {
                    const SvPoint pnt = sv[sv_pos + rank];
                    px = (int)(pnt.pxy & 0xffffu);
                    py = (int)(pnt.pxy >> 16);
                    cr = pix_re(pm, px);
                    ci = pix_im(pm, py);
                    x = pnt.x;
                    y = pnt.y;
                    x2 = __fmul_rn(x, x);
                    y2 = __fmul_rn(y, y);
                    it = (unsigned)PRE;
                    has = true;
                }
                sv_pos += take;
                __syncwarp();
                need = __ballot_sync(FULL, !has);
                continue;
              }
            }
            if (pos >= end) {
                // MANDEL_RF_EXACT: claim no more indices than idle lanes (no index waits in
                // the warp's window behind a long pixel), at the cost of more cursor atomics
                const uint32_t gnow = exact ? min(grab, (uint32_t)__popc(need)) : grab;
                unsigned long long b = 0;
                if (lane == 0)
                    b = atomicAdd(cursor, (unsigned long long)gnow);
                b = __shfl_sync(FULL, b, 0);
                if (b >= total) {
                    exhausted = true;
                    pdl_trigger(pdl_late);
#ifdef MANDEL_RF_TRACE
                    tr_ex = rf_now();
#endif
                    break;
                }
                pos = (uint32_t)b;
                end = (uint32_t)min(b + (unsigned long long)gnow, (unsigned long long)total);
            }
            const unsigned cnt = __popc(need);
            const unsigned avail = end - pos;
            const unsigned take = avail < cnt ? avail : cnt;
            const unsigned rank = __popc(need & lt);
            if (!has && rank < take) {
                map(pos + rank, px, py);
                cr = pix_re(pm, px);
                ci = pix_im(pm, py);
                const float c2 = __fadd_rn(__fmul_rn(cr, cr), __fmul_rn(ci, ci));
                if (c2 <= 3.9f) {
                    has = true;
                    x = y = x2 = y2 = 0.0f;
                    it = 0;
                } else { // per-step loop (escape permanence not guaranteed)
                    sink(px, py, dwell_per_step<K>(cr, ci, maxdwell));
                }
            }
            pos += take;
#ifdef MANDEL_RF_TRACE
            tr_px += take;
#endif
            need = __ballot_sync(FULL, !has);
        }
        const unsigned active = __ballot_sync(FULL, has);
        if (!active)
            break; // cursor exhausted and every lane idle
        // ---------------------------------------------------------------- compute
        // Every lane runs every chunk (no divergent branch); a lane that is parked-to-be
        // (fin) or idle keeps its chunk-start point through predicated selects and its
        // further iterations are discarded.
        const int thresh = exhausted ? 32 : T;
        const bool live = has;
        while (true) {
            const bool keep = fin || !live;
            sx = keep ? sx : x;
            sy = keep ? sy : y;
            sit = keep ? sit : it;
#pragma unroll
            for (int c = 0; c < CKP; ++c) {
#pragma unroll
                for (int k = 0; k < KS; ++k)
                    MANDEL_STEP(x, y, x2, y2, cr, ci);
                if (c < CKP - 1) {
                    ckx[c] = keep ? ckx[c] : x;
                    cky[c] = keep ? cky[c] : y;
                }
            }
            it += K;
            const bool inside = __fadd_rn(x2, y2) <= 4.0f;
            endok = fin ? endok : inside;
            fin = live && (fin || !inside || it >= md);
            const unsigned fm = __ballot_sync(FULL, fin);
            if (fm == active || __popc(fm) >= thresh)
                break;
        }
    }
    // drain the queue
    if (qn > 0)
        replay_batch<KS>(q, qn, pm, md, sink);
#ifdef MANDEL_RF_TRACE
    if (lane == 0 && wrank < 8192 && tslot >= 0 && tslot < 16) {
        g_rf_trace[tslot][wrank][0] = tr_start;
        g_rf_trace[tslot][wrank][1] = tr_ex;
        g_rf_trace[tslot][wrank][2] = rf_now();
        g_rf_trace[tslot][wrank][3] = tr_px | ((unsigned long long)active << 40);
    }
#endif
}


// ============================================================================ packed engine
// Two pixels per lane on the packed FP32 instructions of sm_100 (FMUL2 / FADD2: one issue
// slot drives the FP32 pipe for two lanes' worth of work).  The scalar engine above is
// issue-bound (ncu: 95% of issue slots busy, 27% of them non-FP32 bookkeeping), so halving
// the FP32 issue count lets the bookkeeping of one warp issue while the pipe works on
// another's packed steps.  Each lane owns two independent slots (pixels) whose state lives
// in the two halves of 64-bit register pairs; per slot the algorithm is exactly the scalar
// engine's (same chunked test, parking, bisection replay), with 64 slots per warp.
// mul.rn.f32x2 / add.rn.f32x2 / sub.rn.f32x2 are IEEE RN per half: bit-identical to the
// scalar __fmul_rn / __fadd_rn / __fsub_rn sequence (R4).
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi)
{
    f2_t d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
    return d;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float &lo, float &hi)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b)
{
    f2_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b)
{
    f2_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// Products are fma.rn.f32x2(a, b, -0) = RN(a*b) exactly (x*y + -0 == x*y for every x*y,
// including +-0), with the -0 pair read from constant memory so ptxas cannot see it: ptxas
// 12.9 contracts mul.rn.f32x2 followed by add/sub.rn.f32x2 into FFMA2 even under
// --fmad=false (observed: x*x - y2 fused), which changes the rounding and the dwells.
__constant__ f2_t c_f2_negzero = 0x8000000080000000ull;
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b)
{
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c_f2_negzero));
    return d;
}
// (xy + xy) + ci as one fma.rn.f32x2(xy, {2, 2}, ci) on both halves (R4'; the pair
// of 2.0f from constant memory, like the -0 pair above).
__constant__ f2_t c_f2_two = 0x4000000040000000ull;
__device__ __forceinline__ f2_t f2_fma2x(f2_t xy, f2_t c)
{
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(xy), "l"(c_f2_two), "l"(c));
    return d;
}
// The dwell step of dwell.cuh on both halves (same operation order).
#define MANDEL_STEP2(X, Y, X2, Y2, CR, CI)                                                    \
    do {                                                                                       \
        const f2_t xy_ = f2_mul((X), (Y));                                                     \
        (X) = f2_add(f2_sub((X2), (Y2)), (CR));                                                \
        (Y) = f2_fma2x(xy_, (CI));                                                             \
        (X2) = f2_mul((X), (X));                                                               \
        (Y2) = f2_mul((Y), (Y));                                                               \
    } while (0)

constexpr int RF2_QCAP = 128; // per-warp queue entries (< 64 left over + <= 64 new)

// replay_batch on up to 64 queued points, two per lane (q[lane] low half, q[lane+32] high).
template <int K, class Sink>
__device__ __forceinline__ void replay_batch2(const ParkedPoint *q, int cnt, const PixMap &pm, unsigned md,
                                              Sink &sink)
{
    static_assert((K & (K - 1)) == 0, "K must be a power of two");
    const int lane = threadIdx.x & 31;
    const bool v0 = lane < cnt, v1 = lane + 32 < cnt;
    if (v0) {
        ParkedPoint p0 = q[lane], p1 = p0;
        if (v1)
            p1 = q[lane + 32];
        const f2_t CR = f2_pack(pix_re(pm, p0.px), pix_re(pm, p1.px));
        const f2_t CI = f2_pack(pix_im(pm, p0.py), pix_im(pm, p1.py));
        f2_t BX = f2_pack(p0.x, p1.x), BY = f2_pack(p0.y, p1.y);
        f2_t BX2 = f2_mul(BX, BX), BY2 = f2_mul(BY, BY); // as the chunk start had them
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
            // advance the halves whose first hit lies beyond lo + h
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
        sink(p0.px, p0.py, (int)(lo0 + 1u));
        if (v1)
            sink(p1.px, p1.py, (int)(lo1 + 1u));
    }
    __syncwarp();
}

// Fetch flat index t into one slot: pixel, c, and the zero orbit; pixels with |c|^2 > 3.9
// run the per-step loop here and leave the slot empty.
template <int K, class Map, class Sink>
__device__ __forceinline__ bool rf2_fetch(uint32_t t, const PixMap &pm, int maxdwell, const Map &map, Sink &sink,
                                          int &px, int &py, float &cr, float &ci)
{
    map(t, px, py);
    cr = pix_re(pm, px);
    ci = pix_im(pm, py);
    const float c2 = __fadd_rn(__fmul_rn(cr, cr), __fmul_rn(ci, ci));
    if (c2 <= 3.9f)
        return true;
    sink(px, py, dwell_per_step<K>(cr, ci, maxdwell));
    return false;
}

// Same contract as refill_loop (Map, Sink, cursor, launch shape); q: RF2_QCAP entries.
// T counts parked slots out of the warp's 64.  PRE > 0: short-pixel prepass of PRE steps
// (rf2_prepass above) with the per-warp survivor buffer sv (CH entries; requires
// maxdwell > PRE, else the prepass is off).
template <int K, int T, int CH, class Map, class Sink, int PRE = 0>
__device__ __forceinline__ void refill_loop2(const PixMap &pm, int maxdwell, uint32_t total,
                                             unsigned long long *cursor, const Map &map, Sink &sink,
                                             ParkedPoint *q, int tslot = 0, SvPoint *sv = nullptr,
                                             bool pdl_late = false)
{
    constexpr uint32_t PPL = 8; // pixels per slot before a warp is worth activating
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t min_active = 8u * (uint32_t)c_num_sms;
    uint32_t active = total / (64u * PPL);
    active = active < min_active ? min_active : active;
    active = active > nwarps ? nwarps : active;
    const uint32_t wrank = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    if (wrank >= active)
        return;
#ifdef MANDEL_RF_TRACE
    unsigned long long tr_start = rf_now(), tr_ex = 0, tr_px = 0;
#endif
    uint32_t grab = total / (4u * active);
    grab = grab < 8u ? 8u : (grab > (uint32_t)CH ? (uint32_t)CH : grab);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned md = (unsigned)maxdwell;

    uint32_t pos = 0, end = 0;
    bool exhausted = false;
    int qn = 0;
    // prepass state (warp-uniform)
    bool use_pre = PRE > 0 && maxdwell > PRE && sv != nullptr;
    uint32_t sv_pos = 0, sv_end = 0, pre_tot = 0;
    int pre_esc = 0;

    constexpr int CKP = MANDEL_RF2_CKPT, KS = K / CKP; // sub-chunks (as the scalar engine's CKPT)
    static_assert(CKP >= 1 && K % CKP == 0 && (KS & (KS - 1)) == 0, "RF2_CKPT must split K into powers of two");
    constexpr int NCK = CKP > 1 ? CKP - 1 : 1;
    unsigned sv_it = PRE; // warp-uniform: iteration of the buffered survivors' orbits
    bool has0 = false, has1 = false, fin0 = false, fin1 = false, endok0 = false, endok1 = false;
    int px0 = 0, py0 = 0, px1 = 0, py1 = 0;
    unsigned it0 = 0, it1 = 0, sit0 = 0, sit1 = 0;
    float sx0 = 0.f, sy0 = 0.f, sx1 = 0.f, sy1 = 0.f;
    float ckx0[NCK], cky0[NCK], ckx1[NCK], cky1[NCK];
#pragma unroll
    for (int c = 0; c < NCK; ++c)
        ckx0[c] = cky0[c] = ckx1[c] = cky1[c] = 0.f;
    f2_t X = 0, Y = 0, X2 = 0, Y2 = 0, CR = 0, CI = 0;

    while (true) {
        // ---------------------------------------------------------------- park + refill
        const unsigned f0 = __ballot_sync(FULL, fin0), f1 = __ballot_sync(FULL, fin1);
        if (f0 | f1) {
            // MANDEL_RF_DIRECT: slots that reached maxdwell unescaped get dwell maxdwell
            // without replay
            const bool d0 = MANDEL_RF_DIRECT && fin0 && endok0, d1 = MANDEL_RF_DIRECT && fin1 && endok1;
            if (d0)
                sink(px0, py0, (int)md);
            if (d1)
                sink(px1, py1, (int)md);
            const bool e0 = fin0 && !d0, e1 = fin1 && !d1;
            const unsigned q0 = MANDEL_RF_DIRECT ? __ballot_sync(FULL, e0) : f0;
            const unsigned q1 = MANDEL_RF_DIRECT ? __ballot_sync(FULL, e1) : f1;
            const int n0 = __popc(q0);
            if (e0) {
                ParkedPoint &e = q[qn + __popc(q0 & lt)];
                float bx, by;
                unsigned bit;
                replay_window<CKP, KS>(sx0, sy0, sit0, ckx0, cky0, md, bx, by, bit);
                e.px = px0;
                e.py = py0;
                e.x = bx;
                e.y = by;
                e.it = bit;
            }
            if (e1) {
                ParkedPoint &e = q[qn + n0 + __popc(q1 & lt)];
                float bx, by;
                unsigned bit;
                replay_window<CKP, KS>(sx1, sy1, sit1, ckx1, cky1, md, bx, by, bit);
                e.px = px1;
                e.py = py1;
                e.x = bx;
                e.y = by;
                e.it = bit;
            }
            if (fin0) {
                has0 = false;
                fin0 = false;
            }
            if (fin1) {
                has1 = false;
                fin1 = false;
            }
            qn += n0 + __popc(q1);
            __syncwarp();
            if (qn >= 64) {
                qn -= 64;
                replay_batch2<KS>(q + qn, 64, pm, md, sink);
            }
        }
        unsigned need0 = __ballot_sync(FULL, !has0), need1 = __ballot_sync(FULL, !has1);
        while ((need0 | need1) && !exhausted) {
            if (PRE > 0 && use_pre && sv_pos >= sv_end) {
                // prepass a fresh grab; its survivors refill the buffer.  MANDEL_PRE_SLOTS > 0:
                // at most that many raw pixels per free slot (>= 32), so the survivors -- the
                // long pixels -- do not queue behind busy slots (the exact grabs of §4.6)
                uint32_t gpre = grab;
                if (MANDEL_PRE_SLOTS > 0) {
                    const uint32_t fr = (uint32_t)(__popc(need0) + __popc(need1)) * MANDEL_PRE_SLOTS;
                    gpre = min(grab, fr < 32u ? 32u : fr);
                }
                unsigned long long b = 0;
                if (lane == 0)
                    b = atomicAdd(cursor, (unsigned long long)gpre);
                b = __shfl_sync(FULL, b, 0);
                if (b >= total) {
                    exhausted = true;
                    pdl_trigger(pdl_late);
                    break;
                }
                const uint32_t e = (uint32_t)min(b + (unsigned long long)gpre, (unsigned long long)total);
                sv_pos = 0;
                sv_end = (uint32_t)rf2_prepass<PRE>((uint32_t)b, e, pm, maxdwell, map, sink, sv, pre_esc);
                if constexpr (MANDEL_PRE2 > 0) {
                    // the second stage on every grab's survivors (measured: C3/C4 leaf -3%, C5
                    // +1%; gating it by the first stage's or by its own recent escape fraction
                    // lost most of the C3/C4 gain, profiles/r02_ab_prepass2.jsonl)
                    sv_it = PRE;
                    if (maxdwell > PRE + MANDEL_PRE2 && sv_end > 0) {
                        int esc2 = 0;
                        sv_end = (uint32_t)rf2_prepass_more<PRE, MANDEL_PRE2>(sv, (int)sv_end, pm, sink, esc2);
                        sv_it = PRE + MANDEL_PRE2;
                    }
                }
                pre_tot += e - (uint32_t)b;
                if (pre_tot >= MANDEL_PRE_WINDOW) { // windowed: the list runs hot (long) leaves first
                    use_pre = MANDEL_PRE_MINFRAC * pre_tot <= 100u * (uint32_t)pre_esc;
                    pre_tot = 0;
                    pre_esc = 0;
                }
                continue;
            }
            if (PRE > 0 && sv_pos < sv_end) { // deal survivors (orbit at iteration PRE)
                const unsigned c0 = __popc(need0);
                const unsigned cnt = c0 + __popc(need1);
                const unsigned avail = sv_end - sv_pos;
                const unsigned take = avail < cnt ? avail : cnt;
                const unsigned r0 = __popc(need0 & lt), r1 = c0 + __popc(need1 & lt);
                float cr0, ci0, cr1, ci1, xa0, xa1, ya0, ya1, qa0, qa1, wa0, wa1;
                f2_unpack(CR, cr0, cr1);
                f2_unpack(CI, ci0, ci1);
                f2_unpack(X, xa0, xa1);
                f2_unpack(Y, ya0, ya1);
                f2_unpack(X2, qa0, qa1);
                f2_unpack(Y2, wa0, wa1);
                if (!has0 && r0 < take) {
                    const SvPoint p = sv[sv_pos + r0];
                    px0 = (int)(p.pxy & 0xffffu);
                    py0 = (int)(p.pxy >> 16);
#if MANDEL_SV_C
                    cr0 = p.cr;
                    ci0 = p.ci;
#else
                    cr0 = pix_re(pm, px0);
                    ci0 = pix_im(pm, py0);
#endif
                    qa0 = __fmul_rn(p.x, p.x);
                    wa0 = __fmul_rn(p.y, p.y);
                    xa0 = p.x;
                    ya0 = p.y;
                    it0 = sv_it;
                    has0 = true;
                }
                if (!has1 && r1 < take) {
                    const SvPoint p = sv[sv_pos + r1];
                    px1 = (int)(p.pxy & 0xffffu);
                    py1 = (int)(p.pxy >> 16);
#if MANDEL_SV_C
                    cr1 = p.cr;
                    ci1 = p.ci;
#else
                    cr1 = pix_re(pm, px1);
                    ci1 = pix_im(pm, py1);
#endif
                    qa1 = __fmul_rn(p.x, p.x);
                    wa1 = __fmul_rn(p.y, p.y);
                    xa1 = p.x;
                    ya1 = p.y;
                    it1 = sv_it;
                    has1 = true;
                }
                CR = f2_pack(cr0, cr1);
                CI = f2_pack(ci0, ci1);
                X = f2_pack(xa0, xa1);
                Y = f2_pack(ya0, ya1);
                X2 = f2_pack(qa0, qa1);
                Y2 = f2_pack(wa0, wa1);
                sv_pos += take;
                __syncwarp();
                need0 = __ballot_sync(FULL, !has0);
                need1 = __ballot_sync(FULL, !has1);
                continue;
            }
            if (pos >= end) {
                // MANDEL_RF_EXACT: claim no more indices than idle lanes (no index waits in
                // the warp's window behind a long pixel), at the cost of more cursor atomics
                const uint32_t gnow = MANDEL_RF_EXACT ? min(grab, (uint32_t)(__popc(need0) + __popc(need1))) : grab;
                unsigned long long b = 0;
                if (lane == 0)
                    b = atomicAdd(cursor, (unsigned long long)gnow);
                b = __shfl_sync(FULL, b, 0);
                if (b >= total) {
                    exhausted = true;
                    pdl_trigger(pdl_late);
#ifdef MANDEL_RF_TRACE
                    tr_ex = rf_now();
#endif
                    break;
                }
                pos = (uint32_t)b;
                end = (uint32_t)min(b + (unsigned long long)gnow, (unsigned long long)total);
            }
            const unsigned c0 = __popc(need0);
            const unsigned cnt = c0 + __popc(need1);
            const unsigned avail = end - pos;
            const unsigned take = avail < cnt ? avail : cnt;
            const unsigned r0 = __popc(need0 & lt), r1 = c0 + __popc(need1 & lt);
            float cr0, ci0, cr1, ci1;
            f2_unpack(CR, cr0, cr1);
            f2_unpack(CI, ci0, ci1);
            bool new0 = false, new1 = false;
            if (!has0 && r0 < take)
                new0 = has0 = rf2_fetch<K>(pos + r0, pm, maxdwell, map, sink, px0, py0, cr0, ci0);
            if (!has1 && r1 < take)
                new1 = has1 = rf2_fetch<K>(pos + r1, pm, maxdwell, map, sink, px1, py1, cr1, ci1);
            if (new0 | new1) {
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
#ifdef MANDEL_RF_TRACE
            tr_px += take;
#endif
            if (PRE > 0 && !use_pre && sv != nullptr && maxdwell > PRE) { // retry the prepass later
                pre_tot += take;
                if (pre_tot >= MANDEL_PRE_WINDOW && pos >= end) {
                    use_pre = true;
                    pre_tot = 0;
                }
            }
            need0 = __ballot_sync(FULL, !has0);
            need1 = __ballot_sync(FULL, !has1);
        }
        const unsigned a0m = __ballot_sync(FULL, has0), a1m = __ballot_sync(FULL, has1);
        if (!(a0m | a1m))
            break; // cursor exhausted and every slot idle
        // ---------------------------------------------------------------- compute
        const int thresh = exhausted ? 64 : T;
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
            for (int c = 0; c < CKP; ++c) {
#pragma unroll
                for (int k = 0; k < KS; ++k)
                    MANDEL_STEP2(X, Y, X2, Y2, CR, CI);
                if (c < CKP - 1) {
                    float al, ah, bl, bh;
                    f2_unpack(X, al, ah);
                    f2_unpack(Y, bl, bh);
                    ckx0[c] = keep0 ? ckx0[c] : al;
                    cky0[c] = keep0 ? cky0[c] : bl;
                    ckx1[c] = keep1 ? ckx1[c] : ah;
                    cky1[c] = keep1 ? cky1[c] : bh;
                }
            }
            it0 += K;
            it1 += K;
            float m0, m1;
            f2_unpack(f2_add(X2, Y2), m0, m1);
            const bool in0 = m0 <= 4.0f, in1 = m1 <= 4.0f;
            endok0 = fin0 ? endok0 : in0;
            endok1 = fin1 ? endok1 : in1;
            fin0 = live0 && (fin0 || !in0 || it0 >= md);
            fin1 = live1 && (fin1 || !in1 || it1 >= md);
            const unsigned g0 = __ballot_sync(FULL, fin0), g1 = __ballot_sync(FULL, fin1);
            if ((g0 == a0m && g1 == a1m) || __popc(g0) + __popc(g1) >= thresh)
                break;
        }
    }
    while (qn > 0) { // drain the queue
        const int c = qn < 64 ? qn : 64;
        qn -= c;
        replay_batch2<KS>(q + qn, c, pm, md, sink);
    }
#ifdef MANDEL_RF_TRACE
    if (lane == 0 && wrank < 8192 && tslot >= 0 && tslot < 16) {
        g_rf_trace[tslot][wrank][0] = tr_start;
        g_rf_trace[tslot][wrank][1] = tr_ex;
        g_rf_trace[tslot][wrank][2] = rf_now();
        g_rf_trace[tslot][wrank][3] = tr_px | ((unsigned long long)active << 40);
    }
#endif
}

} // namespace mandel
