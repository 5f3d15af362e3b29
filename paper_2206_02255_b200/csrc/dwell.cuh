// dwell.cuh -- the FP32 Mandelbrot dwell core shared by every sm_100a kernel.
//
// Dwell (Sec. 7): z_{i+1} = z_i^2 + c, z_0 = 0; dwell = first i >= 1 with
// |z_i|^2 > 4, else maxdwell (R2).  Every float operation is an explicit
// round-to-nearest intrinsic (__fmul_rn / __fadd_rn / __fsub_rn / __fmaf_rn), so ptxas can
// never contract a multiply-add into an FFMA and the integer dwell is bit-identical to any
// IEEE binary32 implementation of the operation order of DESIGN.md R4:
//     xy = x*y;  x = (x2 - y2) + cr;  y = (xy + xy) + ci;  x2 = x*x;  y2 = y*y
// with one exact rewrite (R4'): (xy + xy) + ci is computed as fma(xy, 2, ci).  2*xy is exact,
// so the one rounding of the fma is the second addition's; the two differ only if xy + xy
// overflows and |ci| >= 2^103 pulls the sum back -- an orbit that escaped steps earlier, so
// no dwell changes (pinned in tests/native/fma2_identity.c).  3 FMUL + 2 FADD + 1 FFMA
// (immediate form) = 6 FP32 instructions per iteration instead of 7; the x2/y2 products double
// as the next iteration's squares and the escape test's operands.
//
// Iterations run in unrolled chunks of K with ONE escape test per chunk ("!(mag <= 4)",
// so inf/NaN count as escaped).  On a hit the chunk is replayed one step at a time from
// the saved state, which recovers the exact first-escape index.  This is exact because
// escape is permanent when |c| <= 1.975 (|c|^2 <= 3.9 below): once fl(x2+y2) > 4 the
// exact |z| > 2 - 2^-46, so |z'| >= |z|^2 - |c| > 2.02 and |z| then grows monotonically
// until it overflows to inf/NaN.  Pixels with |c|^2 > 3.9 take the
// per-step loop only (they escape within a handful of iterations anyway).
#pragma once
#include <stdint.h>

namespace mandel {

struct PixMap {
    float x0, y0, dx, dy; // (float)re_min, (float)im_min, (float)((re_max-re_min)/n), ...
};

// Pixel-centre sampling (R3): c = x0 + ((float)j + 0.5f) * dx, one RN op each.
__device__ __forceinline__ float pix_re(const PixMap &m, int j)
{
    return __fadd_rn(m.x0, __fmul_rn(__fadd_rn(__int2float_rn(j), 0.5f), m.dx));
}
__device__ __forceinline__ float pix_im(const PixMap &m, int i)
{
    return __fadd_rn(m.y0, __fmul_rn(__fadd_rn(__int2float_rn(i), 0.5f), m.dy));
}

#define MANDEL_STEP(x, y, x2, y2, cr, ci)                                                     \
    do {                                                                                       \
        float xy_ = __fmul_rn((x), (y));                                                       \
        (x) = __fadd_rn(__fsub_rn((x2), (y2)), (cr));                                          \
        (y) = __fmaf_rn(xy_, 2.0f, (ci)); /* == (xy + xy) + ci, R4' */                        \
        (x2) = __fmul_rn((x), (x));                                                            \
        (y2) = __fmul_rn((y), (y));                                                            \
    } while (0)

template <int K>
__device__ __forceinline__ int dwell(float cr, float ci, int maxdwell)
{
    float x = 0.0f, y = 0.0f, x2 = 0.0f, y2 = 0.0f;
    int i = 0;
    const float c2 = __fadd_rn(__fmul_rn(cr, cr), __fmul_rn(ci, ci));
    if (c2 <= 3.9f) {
        const int lim = maxdwell - K;
        while (i <= lim) {
            const float sx = x, sy = y, sx2 = x2, sy2 = y2;
#pragma unroll
            for (int k = 0; k < K; ++k)
                MANDEL_STEP(x, y, x2, y2, cr, ci);
            if (!(__fadd_rn(x2, y2) <= 4.0f)) { // escaped somewhere in this chunk
                x = sx;
                y = sy;
                x2 = sx2;
                y2 = sy2;
                break;
            }
            i += K;
        }
    }
    while (i < maxdwell) { // replay / tail / |c| ~ 2: one escape test per iteration
        MANDEL_STEP(x, y, x2, y2, cr, ci);
        ++i;
        if (__fadd_rn(x2, y2) > 4.0f)
            return i;
    }
    return maxdwell;
}

} // namespace mandel
