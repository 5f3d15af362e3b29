// mandel3d.cu -- libmandel3d.so (include/mandel3d.h): ASK on k = 3 orthotopes (NEXT-4,
// P:549-597).  Same arithmetic as the 2-D path (dwell.cuh: explicit RN FP32
// operations, no FMA, chunked escape test with exact replay), z_0 = w instead of 0.
//
// Per level l (side d): k3_surface computes the dwell of every surface voxel of every region
// (flat grid-stride over count_l * S(d), S(d) = d^3 - (d-2)^3), k3_classify reduces each
// region's surface (block per region) and appends it to the fill list, the next OLT (r^3
// consecutive slots per subdividing region, one atomicAdd, children in canonical order) or
// the leaf list; k3_fill writes the uniform cubes with 128-bit stores; after the last level
// k3_leaf computes the leaves' interior voxels.  Region counts live in the workspace header
// and every kernel reads them there, so a call is a fixed sequence of launches with no host
// round trip.  OLT entries are the canonical-order SFC scalar of the region's corner voxel,
// Omega(p) = (p_z << 2 log n) | (p_y << log n) | p_x (P:585-588 with |G| = n per axis).
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <cstring>

#include "../../include/mandel3d.h"
#include "dwell.cuh"

namespace m3 {

constexpr int MAXL = 16;
constexpr uint32_t MAGIC = 0x4d334b53u; // "M3KS"
constexpr int K = 8;                    // iterations per escape test

struct Hdr {
    uint32_t magic, levels, n, g, r, B, pad[2];
    uint32_t n_subdiv[MAXL], n_fill[MAXL], n_leaf;
    uint32_t pad2;
    unsigned long long border_px[MAXL], border_iters[MAXL], leaf_px, leaf_iters;
};
static_assert(sizeof(Hdr) <= 4096, "header");

struct Axis {
    float x0, y0, z0, dx, dy, dz;
};

// Voxel centre on each axis (reading R16): lo + ((float)k + 0.5f) * step, one RN op each.
__device__ __forceinline__ float vc(float lo, float step, int k)
{
    return __fadd_rn(lo, __fmul_rn(__fadd_rn(__int2float_rn(k), 0.5f), step));
}

// Dwell from z_0 = w (reading R15): dwell.cuh's chunked loop with x = w.
__device__ __forceinline__ int dwell3(float cr, float ci, float w, int maxdwell)
{
    float x = w, y = 0.0f, x2 = __fmul_rn(w, w), y2 = 0.0f;
    int i = 0;
    const float c2 = __fadd_rn(__fmul_rn(cr, cr), __fmul_rn(ci, ci));
    if (c2 <= 3.9f) { // escape is permanent: test once per chunk
        const int lim = maxdwell - K;
        while (i <= lim) {
            const float sx = x, sy = y, sx2 = x2, sy2 = y2;
#pragma unroll
            for (int k = 0; k < K; ++k)
                MANDEL_STEP(x, y, x2, y2, cr, ci);
            if (!(__fadd_rn(x2, y2) <= 4.0f)) {
                x = sx;
                y = sy;
                x2 = sx2;
                y2 = sy2;
                break;
            }
            i += K;
        }
    }
    while (i < maxdwell) {
        MANDEL_STEP(x, y, x2, y2, cr, ci);
        ++i;
        if (__fadd_rn(x2, y2) > 4.0f)
            return i;
    }
    return maxdwell;
}

struct Args {
    Axis ax;
    int maxdwell, logn, level, d, r, g, subdivide, L, n, B;
    int *out;
    Hdr *hdr;
    const uint32_t *olt_in;
    uint32_t *olt_out;
    uint2 *fill; // this level's segment: (Omega, value)
    uint32_t *leaf;
};

__device__ __forceinline__ void unomega(const Args &a, uint32_t o, int &x, int &y, int &z)
{
    const uint32_t m = (1u << a.logn) - 1u;
    x = (int)(o & m);
    y = (int)((o >> a.logn) & m);
    z = (int)(o >> (2 * a.logn));
}
__device__ __forceinline__ uint32_t omega(const Args &a, int x, int y, int z)
{
    return (uint32_t)x | ((uint32_t)y << a.logn) | ((uint32_t)z << (2 * a.logn));
}
__device__ __forceinline__ long long vidx(const Args &a, int x, int y, int z)
{
    return ((long long)z << (2 * a.logn)) + ((long long)y << a.logn) + x;
}

__device__ __forceinline__ uint32_t level_count(const Args &a)
{
    if (a.level == 0)
        return (uint32_t)(a.g * a.g * a.g);
    return (uint32_t)(a.r * a.r * a.r) * *((volatile uint32_t *)&a.hdr->n_subdiv[a.level - 1]);
}

// Surface voxel s in [0, S(d)) of the cube with corner (x0, y0, z0): the z = 0 and z = d-1
// faces (d^2 each), then the 4d-4 ring of each slice 1..d-2 (top row, bottom row, left and
// right columns without their corners).
__device__ __forceinline__ void surface_voxel(long long s, int d, int &x, int &y, int &z)
{
    const long long dd = (long long)d * d;
    if (s < 2 * dd) {
        const int f = (int)(s / dd), q = (int)(s - f * dd);
        z = f ? d - 1 : 0;
        y = q / d;
        x = q - y * d;
        return;
    }
    const long long t = s - 2 * dd;
    const int ring = 4 * d - 4;
    const int zz = (int)(t / ring), b = (int)(t - (long long)zz * ring);
    z = 1 + zz;
    if (b < d) {
        x = b;
        y = 0;
    } else if (b < 2 * d) {
        x = b - d;
        y = d - 1;
    } else if (b < 3 * d - 2) {
        x = 0;
        y = 1 + (b - 2 * d);
    } else {
        x = d - 1;
        y = 1 + (b - (3 * d - 2));
    }
}

__host__ __device__ __forceinline__ long long surface_count(int d)
{
    const long long i = d > 2 ? (long long)(d - 2) : 0;
    return (long long)d * d * d - i * i * i;
}

template <int TPB>
__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, unsigned long long *s)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0)
        s[threadIdx.x >> 5] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < TPB / 32; ++i)
            t += s[i];
    return t;
}

// ------------------------------------------------------------------------------ kernels
__global__ void k3_exhaustive(Axis ax, int n, int maxdwell, int *out)
{
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int z = blockIdx.z;
    if (x >= n || y >= n)
        return;
    const int v = dwell3(vc(ax.x0, ax.dx, x), vc(ax.y0, ax.dy, y), vc(ax.z0, ax.dz, z), maxdwell);
    out[((long long)z * n + y) * n + x] = v;
}

__global__ void k3_init(Args a)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t *hw = reinterpret_cast<uint32_t *>(a.hdr);
    constexpr int words = sizeof(Hdr) / 4;
    for (int w = t; w < words; w += gridDim.x * blockDim.x)
        if (w >= 6) // magic, levels, n, g, r, B are written below
            hw[w] = 0u;
    if (t == 0) {
        a.hdr->magic = MAGIC;
    } else if (t == 1) {
        a.hdr->levels = (uint32_t)a.L;
        a.hdr->n = (uint32_t)a.n;
        a.hdr->g = (uint32_t)a.g;
        a.hdr->r = (uint32_t)a.r;
        a.hdr->B = (uint32_t)a.B;
    }
    const int G = a.g * a.g * a.g;
    for (int k = t; k < G; k += gridDim.x * blockDim.x) {
        const int gx = k % a.g, gy = (k / a.g) % a.g, gz = k / (a.g * a.g);
        const_cast<uint32_t *>(a.olt_in)[k] = omega(a, gx * a.d, gy * a.d, gz * a.d);
    }
}

// Border reuse (as the 2-D B200 scheme): the surfaces of the r^3 children of
// a subdivided parent (side D = r d) are the parent's surface -- already computed, with its
// final dwells in the volume -- plus the interior voxels of the parent lying on a division
// plane (relative coordinate k d - 1 or k d, k = 1..r-1, on some axis).  Per axis the
// a = D-2 interior values split into M = 2(r-1) plane values and N = r(d-2) others, so the new
// voxels are a^3 - N^3 = M a^2 + N M a + N^2 M: x on a plane; x off, y on; x, y off, z on.
__host__ __device__ __forceinline__ long long new_surface_count(int d, int r)
{
    const long long a = (long long)r * d - 2, N = (long long)r * (d - 2);
    return a * a * a - N * N * N;
}
__device__ __forceinline__ int plane_val(int i, int d) { return (i / 2 + 1) * d - 1 + (i & 1); }
__device__ __forceinline__ int off_val(int j, int d) { return (j / (d - 2)) * d + 1 + j % (d - 2); }
__device__ __forceinline__ void new_surface_voxel(long long t, int d, int r, int &x, int &y, int &z)
{
    const long long a = (long long)r * d - 2, M = 2 * (r - 1), N = (long long)r * (d - 2);
    if (t < M * a * a) { // x on a plane, y and z any interior value
        const long long i = t / (a * a), q = t - i * a * a;
        x = plane_val((int)i, d);
        y = 1 + (int)(q / a);
        z = 1 + (int)(q % a);
        return;
    }
    t -= M * a * a;
    if (t < N * M * a) { // x off, y on a plane, z any
        const long long j = t / (M * a), q = t - j * M * a;
        x = off_val((int)j, d);
        y = plane_val((int)(q / a), d);
        z = 1 + (int)(q % a);
        return;
    }
    t -= N * M * a; // x, y off, z on a plane
    const long long j = t / (N * M), q = t - j * N * M;
    x = off_val((int)j, d);
    y = off_val((int)(q / M), d);
    z = plane_val((int)(q % M), d);
}

template <bool STATS>
__global__ void __launch_bounds__(256) k3_surface(Args a)
{
    __shared__ unsigned long long s_sum[8];
    // level 0: the whole surface of every region; level l > 0: the new plane voxels of every
    // region subdivided at level l-1 (its first child's corner is the parent's corner)
    const bool reuse = a.level > 0;
    const long long S = reuse ? new_surface_count(a.d, a.r) : surface_count(a.d);
    const uint32_t units = reuse ? *((volatile uint32_t *)&a.hdr->n_subdiv[a.level - 1]) : level_count(a);
    const long long total = S * (long long)units;
    const uint32_t rrr = (uint32_t)(a.r * a.r * a.r);
    unsigned long long it = 0, px = 0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const uint32_t p = (uint32_t)(t / S);
        int x0, y0, z0, x, y, z;
        unomega(a, a.olt_in[reuse ? p * rrr : p], x0, y0, z0);
        if (reuse)
            new_surface_voxel(t - (long long)p * S, a.d, a.r, x, y, z);
        else
            surface_voxel(t - (long long)p * S, a.d, x, y, z);
        x += x0;
        y += y0;
        z += z0;
        const int v = dwell3(vc(a.ax.x0, a.ax.dx, x), vc(a.ax.y0, a.ax.dy, y), vc(a.ax.z0, a.ax.dz, z), a.maxdwell);
        a.out[vidx(a, x, y, z)] = v;
        if (STATS) {
            it += (unsigned long long)v;
            px += 1;
        }
    }
    if (STATS) {
        it = block_sum<256>(it, s_sum);
        if (threadIdx.x == 0 && it)
            atomicAdd(&a.hdr->border_iters[a.level], it);
        px = block_sum<256>(px, s_sum);
        if (threadIdx.x == 0 && px)
            atomicAdd(&a.hdr->border_px[a.level], px);
    }
}

// Block per region (grid-stride): (min, max) over the surface, then the decision (P:216,
// R17) and the list appends (compact concurrent insertion).
__global__ void __launch_bounds__(256) k3_classify(Args a)
{
    __shared__ int s_lo[8], s_hi[8];
    __shared__ uint32_t s_base;
    const uint32_t count = level_count(a);
    const long long S = surface_count(a.d);
    const int rrr = a.r * a.r * a.r, h = a.d / a.r;
    for (uint32_t ri = blockIdx.x; ri < count; ri += gridDim.x) {
        const uint32_t off = a.olt_in[ri];
        int x0, y0, z0;
        unomega(a, off, x0, y0, z0);
        int lo = INT_MAX, hi = INT_MIN;
        for (long long s = threadIdx.x; s < S; s += blockDim.x) {
            int x, y, z;
            surface_voxel(s, a.d, x, y, z);
            const int v = __ldcg(a.out + vidx(a, x0 + x, y0 + y, z0 + z));
            lo = min(lo, v);
            hi = max(hi, v);
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if ((threadIdx.x & 31) == 0) {
            s_lo[threadIdx.x >> 5] = lo;
            s_hi[threadIdx.x >> 5] = hi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                lo = min(lo, s_lo[w]);
                hi = max(hi, s_hi[w]);
            }
            uint32_t base = UINT_MAX;
            if (lo == hi) {
                const uint32_t e = atomicAdd(&a.hdr->n_fill[a.level], 1u);
                a.fill[e] = make_uint2(off, (uint32_t)lo);
            } else if (a.subdivide) {
                base = atomicAdd(&a.hdr->n_subdiv[a.level], 1u);
            } else {
                a.leaf[atomicAdd(&a.hdr->n_leaf, 1u)] = off;
            }
            s_base = base;
        }
        __syncthreads();
        const uint32_t base = s_base;
        if (base != UINT_MAX)
            for (int c = threadIdx.x; c < rrr; c += blockDim.x) {
                const int cx = c % a.r, cy = (c / a.r) % a.r, cz = c / (a.r * a.r);
                a.olt_out[(size_t)base * rrr + c] = omega(a, x0 + cx * h, y0 + cy * h, z0 + cz * h);
            }
        __syncthreads();
    }
}

// Uniform cubes: flat over all voxels of the level's filled regions; int4 stores along x
// when d % 4 == 0 (rows 16-byte aligned: the volume base is 256-byte aligned and n % 4 == 0).
template <bool VEC>
__global__ void __launch_bounds__(256) k3_fill(Args a)
{
    const unsigned long long count = *((volatile uint32_t *)&a.hdr->n_fill[a.level]);
    const int d = a.d;
    const int lx = VEC ? d / 4 : d; // units per row
    const unsigned long long per = (unsigned long long)lx * d * d;
    const unsigned long long total = count * per;
    for (unsigned long long u = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; u < total;
         u += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long e = u / per;
        const unsigned long long rem = u - e * per;
        const uint2 f = a.fill[e];
        int x0, y0, z0;
        unomega(a, f.x, x0, y0, z0);
        const int ux = (int)(rem % lx), y = (int)((rem / lx) % d), z = (int)(rem / ((unsigned long long)lx * d));
        const int v = (int)f.y;
        if (VEC)
            __stcs(reinterpret_cast<int4 *>(a.out + vidx(a, x0 + 4 * ux, y0 + y, z0 + z)), make_int4(v, v, v, v));
        else
            a.out[vidx(a, x0 + ux, y0 + y, z0 + z)] = v;
    }
}

template <bool STATS>
__global__ void __launch_bounds__(256) k3_leaf(Args a)
{
    __shared__ unsigned long long s_sum[8];
    const int m = a.d - 2;
    const unsigned long long I = m > 0 ? (unsigned long long)m * m * m : 0ull;
    const unsigned long long total = I * *((volatile uint32_t *)&a.hdr->n_leaf);
    unsigned long long it = 0, px = 0;
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long li = t / I;
        const unsigned long long loc = t - li * I;
        int x0, y0, z0;
        unomega(a, a.leaf[li], x0, y0, z0);
        const int x = x0 + 1 + (int)(loc % m), y = y0 + 1 + (int)((loc / m) % m),
                  z = z0 + 1 + (int)(loc / ((unsigned long long)m * m));
        const int v = dwell3(vc(a.ax.x0, a.ax.dx, x), vc(a.ax.y0, a.ax.dy, y), vc(a.ax.z0, a.ax.dz, z), a.maxdwell);
        a.out[vidx(a, x, y, z)] = v;
        if (STATS) {
            it += (unsigned long long)v;
            px += 1;
        }
    }
    if (STATS) {
        it = block_sum<256>(it, s_sum);
        if (threadIdx.x == 0 && it)
            atomicAdd(&a.hdr->leaf_iters, it);
        px = block_sum<256>(px, s_sum);
        if (threadIdx.x == 0 && px)
            atomicAdd(&a.hdr->leaf_px, px);
    }
}

// ------------------------------------------------------------------------------ host
thread_local char g_err[256] = "";

int fail(cudaError_t e, const char *what)
{
    snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
    return 3;
}
#define CK3(call)                                                                              \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return fail(e_, #call);                                                            \
    } while (0)

bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
int lg2(int64_t v)
{
    int k = 0;
    while ((int64_t(1) << k) < v)
        ++k;
    return k;
}
bool valid_grb(int64_t n, int32_t g, int32_t r, int32_t B)
{
    return pow2(n) && n >= 2 && n <= 1024 && pow2(g) && pow2(r) && pow2(B) && r >= 2 && B >= 2 &&
           (int64_t)g * B <= n;
}
bool valid_region(const mandel3d_region &g)
{
    auto fin = [](double v) { return v == v && v < 1e300 && v > -1e300; };
    return fin(g.re_min) && fin(g.re_max) && fin(g.im_min) && fin(g.im_max) && fin(g.w_min) && fin(g.w_max) &&
           g.re_min < g.re_max && g.im_min < g.im_max && g.w_min < g.w_max;
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
size_t a256(size_t v) { return (v + 255) & ~size_t(255); }

struct Layout {
    int L;
    size_t hdr, olt[2], fill, leaf, total;
    size_t cap[MAXL], fill_off[MAXL];
};

bool make_layout(int64_t n, int32_t g, int32_t r, int32_t B, Layout &lay)
{
    if (!valid_grb(n, g, r, B))
        return false;
    lay.L = levels_of(n, g, r, B);
    if (lay.L > MAXL)
        return false;
    size_t c = (size_t)g * g * g, fsum = 0;
    for (int l = 0; l < lay.L; ++l) {
        lay.cap[l] = c;
        lay.fill_off[l] = fsum;
        fsum += c;
        c *= (size_t)r * r * r;
    }
    const size_t capmax = lay.cap[lay.L - 1];
    size_t o = 0;
    lay.hdr = o;
    o += 4096;
    lay.olt[0] = o;
    o = a256(o + capmax * 4);
    lay.olt[1] = o;
    o = a256(o + capmax * 4);
    lay.fill = o;
    o = a256(o + fsum * 8);
    lay.leaf = o;
    o = a256(o + capmax * 4);
    lay.total = o;
    return true;
}

Axis make_axis(const mandel3d_region &reg, int64_t n)
{
    Axis ax;
    ax.x0 = (float)reg.re_min;
    ax.y0 = (float)reg.im_min;
    ax.z0 = (float)reg.w_min;
    ax.dx = (float)((reg.re_max - reg.re_min) / (double)n);
    ax.dy = (float)((reg.im_max - reg.im_min) / (double)n);
    ax.dz = (float)((reg.w_max - reg.w_min) / (double)n);
    return ax;
}

template <typename Kern>
int resident(Kern k, int tpb, size_t cap_blocks)
{
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, tpb, 0) != cudaSuccess || per < 1)
        per = 1;
    size_t gsz = (size_t)per * (sms > 0 ? sms : 1);
    if (cap_blocks < gsz)
        gsz = cap_blocks;
    return (int)(gsz < 1 ? 1 : gsz);
}

} // namespace m3

using namespace m3;

extern "C" {

size_t mandel3d_ask_workspace_bytes(int64_t n, int32_t g, int32_t r, int32_t B)
{
    Layout lay;
    return make_layout(n, g, r, B, lay) ? lay.total : 0;
}

int32_t mandel3d_ask_levels(int64_t n, int32_t g, int32_t r, int32_t B)
{
    return valid_grb(n, g, r, B) ? levels_of(n, g, r, B) : 0;
}

int mandel3d_exhaustive(mandel3d_region reg, int64_t n, int32_t maxdwell, int32_t *d_out, void *stream)
{
    if (!valid_region(reg) || !pow2(n) || n > 1024 || maxdwell < 1 || !d_out)
        return 1;
    const dim3 blk(16, n >= 16 ? 16 : (unsigned)n);
    const dim3 grd((unsigned)((n + 15) / 16), (unsigned)((n + blk.y - 1) / blk.y), (unsigned)n);
    k3_exhaustive<<<grd, blk, 0, (cudaStream_t)stream>>>(make_axis(reg, n), (int)n, maxdwell, d_out);
    CK3(cudaGetLastError());
    return 0;
}

int mandel3d_ask(mandel3d_region reg, int64_t n, int32_t maxdwell, int32_t g, int32_t r, int32_t B, uint32_t flags,
                 int32_t *d_out, void *d_ws, size_t ws_bytes, void *stream)
{
    Layout lay;
    if (!valid_region(reg) || maxdwell < 1 || !d_out || !d_ws || (flags & ~MANDEL3D_FLAG_STATS) ||
        !make_layout(n, g, r, B, lay) || ((uintptr_t)d_ws % 256) != 0 || ((uintptr_t)d_out % 16) != 0)
        return 1;
    if (ws_bytes < lay.total)
        return 2;
    const bool stats = (flags & MANDEL3D_FLAG_STATS) != 0;
    cudaStream_t s = (cudaStream_t)stream;
    char *ws = (char *)d_ws;
    Args a;
    memset(&a, 0, sizeof a);
    a.ax = make_axis(reg, n);
    a.maxdwell = maxdwell;
    a.logn = lg2(n);
    a.r = r;
    a.g = g;
    a.L = lay.L;
    a.n = (int)n;
    a.B = B;
    a.out = d_out;
    a.hdr = (Hdr *)(ws + lay.hdr);
    a.leaf = (uint32_t *)(ws + lay.leaf);
    uint32_t *olt[2] = {(uint32_t *)(ws + lay.olt[0]), (uint32_t *)(ws + lay.olt[1])};
    int d = (int)(n / g);
    a.level = 0;
    a.d = d;
    a.olt_in = olt[0];
    k3_init<<<(g * g * g + 255) / 256 > 4 ? (g * g * g + 255) / 256 : 4, 256, 0, s>>>(a);
    CK3(cudaGetLastError());
    for (int l = 0; l < lay.L; ++l) {
        a.level = l;
        a.d = d;
        a.subdivide = (d / r >= B) ? 1 : 0;
        a.olt_in = olt[l & 1];
        a.olt_out = olt[(l + 1) & 1];
        a.fill = (uint2 *)(ws + lay.fill) + lay.fill_off[l];
        const size_t cap = lay.cap[l];
        const size_t sblocks = (l == 0 ? cap * (size_t)surface_count(d)
                                       : cap / ((size_t)r * r * r) * (size_t)new_surface_count(d, r)) / 256 + 1;
        if (stats)
            k3_surface<true><<<resident(k3_surface<true>, 256, sblocks), 256, 0, s>>>(a);
        else
            k3_surface<false><<<resident(k3_surface<false>, 256, sblocks), 256, 0, s>>>(a);
        CK3(cudaGetLastError());
        k3_classify<<<resident(k3_classify, 256, cap), 256, 0, s>>>(a);
        CK3(cudaGetLastError());
        const bool vec = d % 4 == 0;
        const size_t fblocks = (cap * (size_t)d * d * d / (vec ? 4 : 1) + 255) / 256;
        if (vec)
            k3_fill<true><<<resident(k3_fill<true>, 256, fblocks), 256, 0, s>>>(a);
        else
            k3_fill<false><<<resident(k3_fill<false>, 256, fblocks), 256, 0, s>>>(a);
        CK3(cudaGetLastError());
        if (l + 1 < lay.L)
            d /= r;
    }
    const size_t lblocks = (lay.cap[lay.L - 1] * (size_t)(d > 2 ? d - 2 : 0) * (d > 2 ? d - 2 : 0) *
                                (d > 2 ? d - 2 : 0) + 255) / 256;
    if (lblocks > 0) {
        if (stats)
            k3_leaf<true><<<resident(k3_leaf<true>, 256, lblocks), 256, 0, s>>>(a);
        else
            k3_leaf<false><<<resident(k3_leaf<false>, 256, lblocks), 256, 0, s>>>(a);
        CK3(cudaGetLastError());
    }
    return 0;
}

int mandel3d_ask_last_stats(const void *d_ws, mandel3d_level_stats *h_out, int32_t max_levels, void *stream)
{
    if (!d_ws || (!h_out && max_levels > 0) || max_levels < 0)
        return -1;
    CK3(cudaStreamSynchronize((cudaStream_t)stream));
    Hdr h;
    CK3(cudaMemcpy(&h, d_ws, sizeof h, cudaMemcpyDeviceToHost));
    if (h.magic != MAGIC || h.levels < 1 || h.levels > (uint32_t)MAXL || h.g == 0 || h.r < 2)
        return -1;
    const int L = (int)h.levels;
    int64_t d = (int64_t)h.n / h.g, regions = (int64_t)h.g * h.g * h.g;
    for (int l = 0; l < L && l < max_levels; ++l) {
        mandel3d_level_stats &st = h_out[l];
        st.level = l;
        st.side = (int32_t)d;
        st.regions_in = regions;
        st.filled = h.n_fill[l];
        st.subdivided = h.n_subdiv[l];
        st.leaves = (l == L - 1) ? h.n_leaf : 0;
        st.border_px = (int64_t)h.border_px[l];
        st.border_iters = (int64_t)h.border_iters[l];
        st.leaf_px = (l == L - 1) ? (int64_t)h.leaf_px : 0;
        st.leaf_iters = (l == L - 1) ? (int64_t)h.leaf_iters : 0;
        regions = st.subdivided * h.r * h.r * h.r;
        d /= h.r;
    }
    return L;
}

const char *mandel3d_last_cuda_error(void) { return g_err; }

} // extern "C"
