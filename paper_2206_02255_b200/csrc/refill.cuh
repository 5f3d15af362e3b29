// refill.cuh -- lane-refill dwell engine for the flat B200 kernels.
//
// The pixels a B200 border or leaf kernel computes are a flat index space [0, total) that a
// Map functor turns into image coordinates.  A plain one-thread-per-pixel kernel loses most
// of the FP32 issue slots to divergence: in a warp, dwells range from 1 to maxdwell exactly
// where ASK leaves and borders are (the fractal boundary), and the warp runs as long as its
// slowest lane.  Here every warp is persistent and keeps its 32 lanes busy:
//
//   * a warp grabs CH consecutive indices at a time from a per-launch cursor in the
//     workspace header (one atomicAdd by lane 0) and deals them to its idle lanes in order
//     (ballot + popc rank), so neighbouring pixels run side by side;
//   * the busy lanes iterate in unrolled chunks of K steps (dwell.cuh's 7-op step, one
//     escape test per chunk, saved chunk-start state); a lane whose pixel escaped or reached
//     maxdwell during a chunk freezes (it is masked out of further chunks);
//   * once T lanes are frozen (or every busy lane is), the frozen lanes replay their last
//     chunk one step at a time from the saved state -- this yields the exact first-escape
//     index (escape is permanent) -- store the dwell, and take new pixels.
//
// The image is the same as the plain kernels' (each pixel's dwell is a pure function); only
// which lane computes which pixel, and when, changes.  Pixels with |c|^2 > 3.9 (outside every
// config region) bypass the chunked loop and use the per-step loop at fetch time.
#pragma once
#include "dwell.cuh"

namespace mandel {

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

// Map: __device__ void operator()(unsigned long long t, int &x, int &y) const
// Sink: __device__ void operator()(int x, int y, int v)   (store + optional stats)
template <int K, int T, int CH, class Map, class Sink>
__device__ __forceinline__ void refill_loop(const PixMap &pm, int maxdwell, unsigned long long total,
                                            unsigned long long *cursor, const Map &map, Sink &sink)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;

    unsigned long long pos = 0, end = 0; // warp-uniform chunk window [pos, end)
    bool exhausted = false;              // warp-uniform: the cursor ran past total

    bool has = false, fin = false;
    int px = 0, py = 0;
    float cr = 0.f, ci = 0.f, x = 0.f, y = 0.f, x2 = 0.f, y2 = 0.f;
    float sx = 0.f, sy = 0.f, sx2 = 0.f, sy2 = 0.f;
    unsigned it = 0, sit = 0;
    const unsigned md = (unsigned)maxdwell;

    while (true) {
        // ---------------------------------------------------------------- refill phase
        if (has && fin) { // exact escape index: replay the last chunk one step at a time
            x = sx;
            y = sy;
            x2 = sx2;
            y2 = sy2;
            it = sit;
            int v = maxdwell;
            while (it < md) {
                MANDEL_STEP(x, y, x2, y2, cr, ci);
                ++it;
                if (__fadd_rn(x2, y2) > 4.0f) {
                    v = (int)it;
                    break;
                }
            }
            sink(px, py, v);
            has = false;
        }
        fin = false;
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
                pos = b;
                end = min(b + (unsigned long long)CH, total);
            }
            const unsigned cnt = __popc(need);
            const unsigned long long avail = end - pos;
            const unsigned take = avail < cnt ? (unsigned)avail : cnt;
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
            return; // cursor exhausted and every lane idle
        // ---------------------------------------------------------------- compute phase
        const int thresh = exhausted ? 32 : T;
        while (true) {
            if (has && !fin) {
                sx = x;
                sy = y;
                sx2 = x2;
                sy2 = y2;
                sit = it;
#pragma unroll
                for (int k = 0; k < K; ++k)
                    MANDEL_STEP(x, y, x2, y2, cr, ci);
                it += K;
                fin = !(__fadd_rn(x2, y2) <= 4.0f) || it >= md;
            }
            const unsigned f = __ballot_sync(FULL, fin);
            if (f == active || __popc(f) >= thresh)
                break;
        }
    }
}

} // namespace mandel
