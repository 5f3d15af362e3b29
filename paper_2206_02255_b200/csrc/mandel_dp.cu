// mandel_dp.cu -- the paper's Dynamic Parallelism baseline (include/mandel_dp.h): recursive
// Mariani-Silver with CUDA Dynamic Parallelism (CDP2, device-side launches into the
// fire-and-forget stream), one block per region (SBR), one child grid per subdividing node
// ("one kernel per node of the subdivision tree").  Built with -rdc=true into its own
// library (libmandel_dp.so) so that relocatable device code does not touch the ASK kernels.
//
// P:NNN = /root/reference/PAPER.md line NNN.
#include <climits>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/mandel_dp.h"
#include "dwell.cuh"

namespace mandel {
namespace dp {

constexpr int DWELL_K = 8; // iterations per escape test (dwell.cuh, exact replay)

struct DpArgs {
    PixMap map;
    int maxdwell;
    long long pitch;
    int *out;
    int r, B;
    int vec; // out 16-byte aligned and pitch % 4 == 0: 128-bit fill stores
};

// Border pixel b in [0, 4d-4): top row, bottom row, left and right columns without corners.
__device__ __forceinline__ void ring_xy(int b, int d, int x0, int y0, int &x, int &y)
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

template <int TPB>
__global__ void k_dp(DpArgs a, int bx, int by, int d);

// One child grid of r x r blocks on the sub-regions of side s of the region at (x0, y0)
// (block size from the child's ring length, like the ASK-SBR level kernels).
__device__ __forceinline__ void launch_children(const DpArgs &a, int x0, int y0, int s)
{
    const dim3 grid(a.r, a.r);
    if (4 * s - 4 >= 256)
        k_dp<256><<<grid, 256, 0, cudaStreamFireAndForget>>>(a, x0, y0, s);
    else
        k_dp<128><<<grid, 128, 0, cudaStreamFireAndForget>>>(a, x0, y0, s);
}

// One block per region: block (bx_i, by_i) of the grid handles the region of side d at
// (bx + blockIdx.x d, by + blockIdx.y d).  Border Q, then fill T / child launch / leaf L.
template <int TPB>
__global__ void __launch_bounds__(TPB) k_dp(DpArgs a, int bx, int by, int d)
{
    __shared__ int s_lo[TPB / 32], s_hi[TPB / 32];
    const int x0 = bx + (int)blockIdx.x * d, y0 = by + (int)blockIdx.y * d;
    const int ring = 4 * d - 4;
    int lo = INT_MAX, hi = INT_MIN;
    for (int b = threadIdx.x; b < ring; b += TPB) {
        int x, y;
        ring_xy(b, d, x0, y0, x, y);
        const int v = dwell<DWELL_K>(pix_re(a.map, x), pix_im(a.map, y), a.maxdwell);
        a.out[(long long)y * a.pitch + x] = v;
        lo = min(lo, v);
        hi = max(hi, v);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_lo[w] = lo;
        s_hi[w] = hi;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < TPB / 32; ++i) {
        lo = min(lo, s_lo[i]);
        hi = max(hi, s_hi[i]);
    }
    if (lo == hi) { // uniform border: terminal work, the block fills the region
        if (a.vec && d % 4 == 0) {
            const int q = d >> 2;
            const int4 v4 = make_int4(lo, lo, lo, lo);
            for (int t = threadIdx.x; t < d * q; t += TPB) {
                const int row = t / q, c = t - row * q;
                __stcs(reinterpret_cast<int4 *>(a.out + (long long)(y0 + row) * a.pitch + x0) + c, v4);
            }
        } else {
            for (int t = threadIdx.x; t < d * d; t += TPB) {
                const int row = t / d, c = t - row * d;
                a.out[(long long)(y0 + row) * a.pitch + x0 + c] = lo;
            }
        }
    } else if (d / a.r >= a.B) { // subdivide: one child grid per node
        if (threadIdx.x == 0)
            launch_children(a, x0, y0, d / a.r);
    } else { // leaf: the block computes the interior
        const int m = d - 2;
        for (int p = threadIdx.x; p < m * m; p += TPB) {
            const int x = x0 + 1 + p % m, y = y0 + 1 + p / m;
            a.out[(long long)y * a.pitch + x] = dwell<DWELL_K>(pix_re(a.map, x), pix_im(a.map, y), a.maxdwell);
        }
    }
}

thread_local char g_err[256] = "";

int fail(cudaError_t e, const char *what)
{
    snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
    return MANDEL_ECUDA;
}

bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

bool valid(const mandel_region &g, int64_t n, int32_t maxdwell, int32_t gg, int32_t r, int32_t B,
           const int32_t *out, int64_t pitch)
{
    auto fin = [](double v) { return v == v && v < 1e300 && v > -1e300; };
    return fin(g.re_min) && fin(g.re_max) && fin(g.im_min) && fin(g.im_max) && g.re_min < g.re_max &&
           g.im_min < g.im_max && pow2(n) && n <= 65536 && pow2(gg) && pow2(r) && pow2(B) && r >= 2 && B >= 2 &&
           (int64_t)gg * B <= n && maxdwell >= 1 && out && pitch >= n;
}

} // namespace dp
} // namespace mandel

using namespace mandel;
using namespace mandel::dp;

extern "C" {

int64_t mandel_dp_pending_launches(int64_t n, int32_t g, int32_t r, int32_t B)
{
    if (!pow2(n) || n > 65536 || !pow2(g) || !pow2(r) || !pow2(B) || r < 2 || B < 2 || (int64_t)g * B > n)
        return 0;
    int64_t d = n / g, nodes = (int64_t)g * g, total = 0;
    while (d / r >= B) { // every region of a subdividing level may launch one child grid
        total += nodes;
        nodes *= (int64_t)r * r;
        d /= r;
    }
    return total;
}

int mandel_dp(mandel_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B, int32_t *d_out,
              int64_t out_pitch, void *stream)
{
    if (!valid(reg, n, maxdwell, g, r, B, d_out, out_pitch))
        return MANDEL_EINVAL;
    const int64_t need = mandel_dp_pending_launches(n, g, r, B);
    size_t cur = 0;
    cudaError_t e = cudaDeviceGetLimit(&cur, cudaLimitDevRuntimePendingLaunchCount);
    if (e != cudaSuccess)
        return fail(e, "cudaDeviceGetLimit(PendingLaunchCount)");
    if ((int64_t)cur < need + 64) {
        e = cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, (size_t)need + 64);
        if (e != cudaSuccess)
            return fail(e, "cudaDeviceSetLimit(PendingLaunchCount)");
    }
    DpArgs a;
    a.map.x0 = (float)reg.re_min;
    a.map.y0 = (float)reg.im_min;
    a.map.dx = (float)((reg.re_max - reg.re_min) / (double)n);
    a.map.dy = (float)((reg.im_max - reg.im_min) / (double)n);
    a.maxdwell = maxdwell;
    a.pitch = out_pitch;
    a.out = d_out;
    a.r = r;
    a.B = B;
    a.vec = ((uintptr_t)d_out % 16 == 0 && out_pitch % 4 == 0) ? 1 : 0;
    const int d0 = (int)(n / g);
    cudaStream_t s = (cudaStream_t)stream;
    if (4 * d0 - 4 >= 256)
        k_dp<256><<<dim3(g, g), 256, 0, s>>>(a, 0, 0, d0);
    else
        k_dp<128><<<dim3(g, g), 128, 0, s>>>(a, 0, 0, d0);
    e = cudaGetLastError();
    if (e != cudaSuccess)
        return fail(e, "k_dp launch");
    return MANDEL_OK;
}

const char *mandel_dp_last_cuda_error(void) { return g_err; }

} // extern "C"
