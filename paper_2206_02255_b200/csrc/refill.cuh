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

// A parked chunk-start point awaiting its exact replay.
struct ParkedPoint {
    int px, py;
    float x, y;
    unsigned it;
};

constexpr int RF_QCAP = 64; // per-warp queue entries (< 32 left over + < 32 new)

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

// Map: __device__ void operator()(uint32_t t, int &x, int &y) const      (t < 2^32)
// Sink: __device__ void operator()(int x, int y, int v)                   (store + stats)
// q: this warp's RF_QCAP-entry queue in shared memory.
// The grab size adapts to the launch: at most CH, but small enough that every warp of the
// grid gets about 4 grabs (small levels -- e.g. one rank's share of a multi-GPU run -- would
// otherwise leave most warps idle while a few run whole grabs of maxdwell pixels), and >= 8.
template <int K, int T, int CH, class Map, class Sink>
__device__ __forceinline__ void refill_loop(const PixMap &pm, int maxdwell, uint32_t total,
                                            unsigned long long *cursor, const Map &map, Sink &sink,
                                            ParkedPoint *q, int tslot = 0)
{
    // Active warps: a launch with few pixels per lane runs like a thread-per-pixel kernel
    // (every warp waits for its slowest lane and there is nothing to refill from), so only
    // ~total/(32*PPL) warps work -- but never fewer than 2 per SM sub-partition (592 on
    // B200), below which one warp per scheduler is latency-bound.  Warp w of block b has
    // rank w*gridDim+b, so the active warps spread over all SMs.  (Idle warps return here and
    // still reach the caller's block-wide reductions.)
    constexpr uint32_t PPL = 8;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t min_active = 8u * (uint32_t)c_num_sms;
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
    grab = grab < 8u ? 8u : (grab > (uint32_t)CH ? (uint32_t)CH : grab);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned md = (unsigned)maxdwell;

    uint32_t pos = 0, end = 0; // warp-uniform chunk window [pos, end)
    bool exhausted = false;    // warp-uniform: the cursor ran past total
    int qn = 0;                // warp-uniform queue fill

    bool has = false, fin = false;
    int px = 0, py = 0;
    float cr = 0.f, ci = 0.f, x = 0.f, y = 0.f, x2 = 0.f, y2 = 0.f, sx = 0.f, sy = 0.f;
    unsigned it = 0, sit = 0;

    while (true) {
        // ---------------------------------------------------------------- park + refill
        const unsigned f = __ballot_sync(FULL, fin);
        if (f) {
            if (fin) {
                ParkedPoint &e = q[qn + __popc(f & lt)];
                e.px = px;
                e.py = py;
                e.x = sx;
                e.y = sy;
                e.it = sit;
                has = false;
                fin = false;
            }
            qn += __popc(f);
            __syncwarp();
            if (qn >= 32) {
                qn -= 32;
                replay_batch<K>(q + qn, 32, pm, md, sink);
            }
        }
        unsigned need = __ballot_sync(FULL, !has);
        while (need && !exhausted) {
            if (pos >= end) {
                unsigned long long b = 0;
                if (lane == 0)
                    b = atomicAdd(cursor, (unsigned long long)grab);
                b = __shfl_sync(FULL, b, 0);
                if (b >= total) {
                    exhausted = true;
#ifdef MANDEL_RF_TRACE
                    tr_ex = rf_now();
#endif
                    break;
                }
                pos = (uint32_t)b;
                end = (uint32_t)min(b + (unsigned long long)grab, (unsigned long long)total);
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
            for (int k = 0; k < K; ++k)
                MANDEL_STEP(x, y, x2, y2, cr, ci);
            it += K;
            fin = live && (fin || !(__fadd_rn(x2, y2) <= 4.0f) || it >= md);
            const unsigned fm = __ballot_sync(FULL, fin);
            if (fm == active || __popc(fm) >= thresh)
                break;
        }
    }
    // drain the queue
    if (qn > 0)
        replay_batch<K>(q, qn, pm, md, sink);
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
