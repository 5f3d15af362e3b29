// refill.cuh -- lane-refill dwell engine for the flat B200 kernels.
//
// The pixels a B200 border or leaf kernel computes are a flat index space [0, total) that a
// Map functor turns into image coordinates.  A plain one-thread-per-pixel kernel loses most
// of the FP32 issue slots to divergence: in a warp, dwells range from 1 to maxdwell exactly
// where ASK leaves and borders are (the fractal boundary: median dwell ~10, 10-20% of the
// pixels at maxdwell), and the warp runs as long as its slowest lane.  Here every warp is
// persistent and keeps its 32 lanes busy:
//
//   * a warp grabs CH consecutive indices at a time from a per-launch cursor in the
//     workspace header (one atomicAdd by lane 0) and deals them to its idle lanes in order
//     (ballot + popc rank), so neighbouring pixels run side by side;
//   * busy lanes iterate in unrolled chunks of K steps (dwell.cuh's 7-op step) with one
//     escape test per chunk, keeping the chunk-start point (x, y, iteration);
//   * a lane whose pixel escaped (or reached maxdwell) during the chunk parks that
//     chunk-start point in a per-warp queue in shared memory and is refilled at once, as
//     soon as T lanes are parked;
//   * whenever 32 points are queued the warp replays them together, one lane each: one
//     step at a time from the chunk start, which yields the exact first-escape index
//     (escape is permanent), then stores the dwell.  Replays thus run with
//     all 32 lanes busy instead of stalling the warp once per escaping lane.
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

// Replay the queued points q[0..cnt) (cnt <= 32), one per lane, and store their dwells.
template <class Sink>
__device__ __forceinline__ void replay_batch(const ParkedPoint *q, int cnt, const PixMap &pm, unsigned md,
                                             int maxdwell, Sink &sink)
{
    const int lane = threadIdx.x & 31;
    if (lane < cnt) {
        const ParkedPoint p = q[lane];
        const float cr = pix_re(pm, p.px), ci = pix_im(pm, p.py);
        float x = p.x, y = p.y;
        float x2 = __fmul_rn(x, x), y2 = __fmul_rn(y, y); // as the chunk start had them
        unsigned it = p.it;
        int v = maxdwell;
        while (it < md) {
            MANDEL_STEP(x, y, x2, y2, cr, ci);
            ++it;
            if (__fadd_rn(x2, y2) > 4.0f) {
                v = (int)it;
                break;
            }
        }
        sink(p.px, p.py, v);
    }
    __syncwarp();
}

// Map: __device__ void operator()(uint32_t t, int &x, int &y) const      (t < 2^32)
// Sink: __device__ void operator()(int x, int y, int v)                   (store + stats)
// q: this warp's RF_QCAP-entry queue in shared memory.
template <int K, int T, int CH, class Map, class Sink>
__device__ __forceinline__ void refill_loop(const PixMap &pm, int maxdwell, uint32_t total,
                                            unsigned long long *cursor, const Map &map, Sink &sink,
                                            ParkedPoint *q)
{
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
                replay_batch(q + qn, 32, pm, md, maxdwell, sink);
            }
        }
        unsigned need = __ballot_sync(FULL, !has);
        while (need && !exhausted) {
            if (pos >= end) {
                unsigned long long b = 0;
                if (lane == 0)
                    b = atomicAdd(cursor, (unsigned long long)CH);
                b = __shfl_sync(FULL, b, 0);
                if (b >= total) {
                    exhausted = true;
                    break;
                }
                pos = (uint32_t)b;
                end = (uint32_t)min(b + (unsigned long long)CH, (unsigned long long)total);
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
        replay_batch(q, qn, pm, md, maxdwell, sink);
}

} // namespace mandel
