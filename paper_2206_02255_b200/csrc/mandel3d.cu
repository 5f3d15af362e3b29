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
#include "refill.cuh" // FastDiv: 32-bit multiply-high division by host-computed magics

using mandel::FastDiv;
using mandel::fdiv;
using mandel::make_fastdiv;

namespace m3 {

constexpr int MAXL = 16;
constexpr uint32_t MAGIC = 0x4d334b53u; // "M3KS"
constexpr int K = 8;                    // iterations per escape test

struct Hdr {
    uint32_t magic, levels, n, g, r, B, pad[2];
    uint32_t n_subdiv[MAXL], n_fill[MAXL], n_leaf;
    uint32_t pad2;
    unsigned long long border_px[MAXL], border_iters[MAXL], leaf_px, leaf_iters;
    unsigned long long cursor[MAXL + 1]; // lane-refill work cursors: surface level l, leaves
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
    // index maps (every flat index space of a call is < n^3 <= 2^30): the level's surface-kernel
    // unit S, d^2, d, the ring 4d-4; for the division planes a^2, a, M a, N M, M (a = r d - 2,
    // M = 2(r-1), N = r(d-2)); the leaf interior side m = d-2 and m^3
    FastDiv fS, fdd, fd, fring, fa2, fa, fMa, fNM, fM, fm, fI;
    int log_d, log_fill_per, log_fill_row; // fill: d, units per cube, units per row (powers of 2)
    // x-boundary planes, transposed (the 3-D colT): every voxel with
    // x mod u in {0, u-1} (u = leaf side; every region's x-faces lie there) is also stored at
    // colT[((2 (x / u) + (x mod u != 0)) * n + z) * n + y], so classification reads the
    // surface's x-columns as runs along y instead of one 32-byte sector per voxel
    int *colT; // NULL: off (u < 8)
    int log_u;
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

__device__ __forceinline__ long long colT_idx(const Args &a, int x, int y, int z)
{
    const int m = x & ((1 << a.log_u) - 1);
    const long long plane = 2 * (x >> a.log_u) + (m != 0);
    return (((plane << a.logn) + z) << a.logn) + y;
}
// A surface voxel's dwell: the volume, plus the transposed x-plane copy when x is on one.
__device__ __forceinline__ void store_surface(const Args &a, int x, int y, int z, int v)
{
    a.out[vidx(a, x, y, z)] = v;
    if (a.colT) {
        const int m = x & ((1 << a.log_u) - 1);
        if (m == 0 || m == (1 << a.log_u) - 1)
            a.colT[colT_idx(a, x, y, z)] = v;
    }
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
__device__ __forceinline__ void surface_voxel(const Args &a, uint32_t s, int &x, int &y, int &z)
{
    const int d = a.d;
    const uint32_t dd = a.fdd.d;
    if (s < 2u * dd) {
        const uint32_t f = s >= dd ? 1u : 0u, q = s - f * dd;
        z = f ? d - 1 : 0;
        y = (int)fdiv(q, a.fd);
        x = (int)q - y * d;
        return;
    }
    const uint32_t t = s - 2u * dd;
    const uint32_t zz = fdiv(t, a.fring);
    const int b = (int)(t - zz * a.fring.d);
    z = 1 + (int)zz;
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

// ------------------------------------------------------------------------------ lane refill
// The 2-D lane-refill engine (refill.cuh) for voxels: persistent warps grab
// flat indices from a per-launch cursor and deal them to idle lanes; busy lanes run K-step
// chunks with one escape test per chunk; a finished lane parks its chunk-start point and is
// refilled once T lanes are parked; 32 parked points are replayed together by bisection over
// the chunk.  A voxel is identified by its SFC scalar Omega (x | y << logn | z << 2 logn).
constexpr int RK = 16, RT = 8, RCH = 64, RTPB = 256, RMINB = 4;
__constant__ int c3_sms;

struct Park3 {
    uint32_t o;
    float x, y;
    unsigned it;
};

__device__ __forceinline__ void voxel_c(const Args &a, uint32_t o, float &cr, float &ci, float &w)
{
    int x, y, z;
    unomega(a, o, x, y, z);
    cr = vc(a.ax.x0, a.ax.dx, x);
    ci = vc(a.ax.y0, a.ax.dy, y);
    w = vc(a.ax.z0, a.ax.dz, z);
}

__device__ __forceinline__ int dwell3_per_step(float cr, float ci, float w, int maxdwell)
{
    float x = w, y = 0.0f, x2 = __fmul_rn(w, w), y2 = 0.0f;
    for (int i = 1; i <= maxdwell; ++i) {
        MANDEL_STEP(x, y, x2, y2, cr, ci);
        if (__fadd_rn(x2, y2) > 4.0f)
            return i;
    }
    return maxdwell;
}

template <bool STATS, bool SURFACE = true>
struct Sink3 {
    const Args *a;
    unsigned long long iters, px;
    __device__ __forceinline__ void operator()(uint32_t o, int v)
    {
        int x, y, z;
        unomega(*a, o, x, y, z);
        if (SURFACE)
            store_surface(*a, x, y, z, v);
        else
            a->out[vidx(*a, x, y, z)] = v;
        if (STATS) {
            iters += (unsigned long long)v;
            px += 1;
        }
    }
};

// Replay q[0..cnt) (cnt <= 32), one per lane: bisection over the K steps after the chunk start
// for the first step where "escaped, or iteration >= maxdwell" holds (monotone, §3.2).
template <class Sink>
__device__ __forceinline__ void replay3(const Args &a, const Park3 *q, int cnt, unsigned md, Sink &sink)
{
    const int lane = threadIdx.x & 31;
    if (lane < cnt) {
        const Park3 p = q[lane];
        float cr, ci, w;
        voxel_c(a, p.o, cr, ci, w);
        float bx = p.x, by = p.y, bx2 = __fmul_rn(bx, bx), by2 = __fmul_rn(by, by);
        unsigned lo = p.it;
#pragma unroll
        for (int h = RK / 2; h >= 1; h /= 2) {
            float x = bx, y = by, x2 = bx2, y2 = by2;
#pragma unroll
            for (int k = 0; k < h; ++k)
                MANDEL_STEP(x, y, x2, y2, cr, ci);
            const bool hit = !(__fadd_rn(x2, y2) <= 4.0f) || lo + (unsigned)h >= md;
            if (!hit) {
                bx = x;
                by = y;
                bx2 = x2;
                by2 = y2;
                lo += (unsigned)h;
            }
        }
        sink(p.o, (int)(lo + 1u));
    }
    __syncwarp();
}

// Map: __device__ uint32_t operator()(unsigned long long t) const -> Omega of flat index t.
template <class Map, class Sink>
__device__ __forceinline__ void refill3(const Args &a, unsigned long long total, unsigned long long *cursor,
                                        const Map &map, Sink &sink, Park3 *q)
{
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const unsigned long long min_active = 8ull * (unsigned long long)c3_sms;
    unsigned long long act = total / (32ull * 8ull);
    act = act < min_active ? min_active : act;
    act = act > nwarps ? nwarps : act;
    const uint32_t wrank = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    if (wrank >= act)
        return;
    unsigned long long grab = total / (4ull * act);
    grab = grab < 8ull ? 8ull : (grab > (unsigned long long)RCH ? (unsigned long long)RCH : grab);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned md = (unsigned)a.maxdwell;
    unsigned long long pos = 0, end = 0;
    bool exhausted = false;
    int qn = 0;
    bool has = false, fin = false;
    uint32_t o = 0;
    float cr = 0.f, ci = 0.f, x = 0.f, y = 0.f, x2 = 0.f, y2 = 0.f, sx = 0.f, sy = 0.f;
    unsigned it = 0, sit = 0;
    while (true) {
        const unsigned f = __ballot_sync(FULL, fin);
        if (f) {
            if (fin) {
                Park3 &e = q[qn + __popc(f & lt)];
                e.o = o;
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
                replay3(a, q + qn, 32, md, sink);
            }
        }
        unsigned need = __ballot_sync(FULL, !has);
        while (need && !exhausted) {
            if (pos >= end) {
                unsigned long long b = 0;
                if (lane == 0)
                    b = atomicAdd(cursor, grab);
                b = __shfl_sync(FULL, b, 0);
                if (b >= total) {
                    exhausted = true;
                    break;
                }
                pos = b;
                end = b + grab < total ? b + grab : total;
            }
            const unsigned cnt = __popc(need);
            const unsigned avail = (unsigned)(end - pos);
            const unsigned take = avail < cnt ? avail : cnt;
            const unsigned rank = __popc(need & lt);
            if (!has && rank < take) {
                o = map(pos + rank);
                float w;
                voxel_c(a, o, cr, ci, w);
                const float c2 = __fadd_rn(__fmul_rn(cr, cr), __fmul_rn(ci, ci));
                if (c2 <= 3.9f) {
                    has = true;
                    x = w;
                    y = 0.0f;
                    x2 = __fmul_rn(w, w);
                    y2 = 0.0f;
                    it = 0;
                } else {
                    sink(o, dwell3_per_step(cr, ci, w, a.maxdwell));
                }
            }
            pos += take;
            need = __ballot_sync(FULL, !has);
        }
        const unsigned active = __ballot_sync(FULL, has);
        if (!active)
            break;
        const int thresh = exhausted ? 32 : RT;
        const bool live = has;
        while (true) {
            const bool keep = fin || !live;
            sx = keep ? sx : x;
            sy = keep ? sy : y;
            sit = keep ? sit : it;
#pragma unroll
            for (int k = 0; k < RK; ++k)
                MANDEL_STEP(x, y, x2, y2, cr, ci);
            it += RK;
            fin = live && (fin || !(__fadd_rn(x2, y2) <= 4.0f) || it >= md);
            const unsigned fm = __ballot_sync(FULL, fin);
            if (fm == active || __popc(fm) >= thresh)
                break;
        }
    }
    if (qn > 0)
        replay3(a, q, qn, md, sink);
}

// ---------------------------------------------------------------- packed lane refill (leaves)
// The 2-D leaf engine (refill.cuh refill_loop2) for voxels: two slots per lane
// stepped with FFMA2/FADD2 (the opaque -0 product of refill.cuh keeps every operation an
// RN single op), T counted out of 64 slots, replay in batches of 64, and the short-voxel
// prepass (PRE steps with a test after every step) on each grab.  Same result per voxel.
using mandel::f2_t;
using mandel::f2_pack;
using mandel::f2_unpack;
using mandel::f2_add;
using mandel::f2_sub;
using mandel::f2_mul;
using mandel::f2_fma2x;
#ifndef MANDEL3D_PK
#define MANDEL3D_PK 32 // packed voxel engine: steps per escape test (16: V2 27.95 ms, 32: 27.53 ms)
#endif
constexpr int PK = MANDEL3D_PK, PT = 8, PCH = 128, PPRE = 16, PMINB = 3;
#ifndef MANDEL3D_PRE_COUNT
#define MANDEL3D_PRE_COUNT 1 // prepass escape test: 0 latch the first escape, 1 float count
#endif
#ifndef MANDEL3D_PRE2
#define MANDEL3D_PRE2 16 // second prepass stage on the survivors (steps; 0: none)
#endif

template <class Sink>
__device__ __forceinline__ void replay3_2(const Args &a, const Park3 *q, int cnt, unsigned md, Sink &sink)
{
    const int lane = threadIdx.x & 31;
    const bool v0 = lane < cnt, v1 = lane + 32 < cnt;
    if (v0) {
        Park3 p0 = q[lane], p1 = p0;
        if (v1)
            p1 = q[lane + 32];
        float cr0, ci0, w0, cr1, ci1, w1;
        voxel_c(a, p0.o, cr0, ci0, w0);
        voxel_c(a, p1.o, cr1, ci1, w1);
        const f2_t CR = f2_pack(cr0, cr1), CI = f2_pack(ci0, ci1);
        f2_t BX = f2_pack(p0.x, p1.x), BY = f2_pack(p0.y, p1.y);
        f2_t BX2 = f2_mul(BX, BX), BY2 = f2_mul(BY, BY);
        unsigned lo0 = p0.it, lo1 = p1.it;
#pragma unroll
        for (int h = PK / 2; h >= 1; h /= 2) {
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
        sink(p0.o, (int)(lo0 + 1u));
        if (v1)
            sink(p1.o, (int)(lo1 + 1u));
    }
    __syncwarp();
}

// Prepass of flat indices [b, e): PPRE steps per voxel with a test after every step; escaped
// voxels are stored, survivors go to sv (orbit at iteration PPRE).  Returns the survivor count.
template <class Map, class Sink>
__device__ __forceinline__ int prepass3(const Args &a, uint32_t b, uint32_t e, const Map &map, Sink &sink, Park3 *sv)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int m = 0;
    for (uint32_t r0 = b; r0 < e; r0 += 32) {
        const uint32_t t = r0 + (uint32_t)lane;
        bool surv = false;
        uint32_t o = 0;
        float x = 0.f, y = 0.f;
        if (t < e) {
            o = map(t);
            float cr, ci, w;
            voxel_c(a, o, cr, ci, w);
            if (__fadd_rn(__fmul_rn(cr, cr), __fmul_rn(ci, ci)) <= 3.9f) {
                x = w;
                float x2 = __fmul_rn(w, w), y2 = 0.f;
#if MANDEL3D_PRE_COUNT
                // the 2-D leaf prepass's counted test (refill.cuh): escape is permanent, so the
                // steps still inside are the steps before the dwell
                float inf_ = 0.0f;
#pragma unroll
                for (int k = 1; k <= PPRE; ++k) {
                    MANDEL_STEP(x, y, x2, y2, cr, ci);
                    inf_ = __fadd_rn(inf_, __fadd_rn(x2, y2) <= 4.0f ? 1.0f : 0.0f);
                }
                const int in_ = (int)inf_;
                const int dw = in_ < PPRE ? in_ + 1 : 0;
#else
                int dw = 0;
#pragma unroll
                for (int k = 1; k <= PPRE; ++k) {
                    MANDEL_STEP(x, y, x2, y2, cr, ci);
                    dw = (dw == 0 && !(__fadd_rn(x2, y2) <= 4.0f)) ? k : dw;
                }
#endif
                if (dw)
                    sink(o, dw);
                else
                    surv = true;
            } else {
                sink(o, dwell3_per_step(cr, ci, w, a.maxdwell));
            }
        }
        const unsigned sm = __ballot_sync(FULL, surv);
        if (surv) {
            Park3 &q = sv[m + __popc(sm & lt)];
            q.o = o;
            q.x = x;
            q.y = y;
            q.it = (unsigned)PPRE;
        }
        m += __popc(sm);
    }
    __syncwarp();
    return m;
}

// Second prepass stage (MANDEL3D_PRE2 = S2 > 0, as refill.cuh rf2_prepass_more): the
// survivors in sv[0, m) run S2 more counted steps, one per lane; escaped voxels are stored,
// the rest compacted in place with their iteration advanced.  Returns the survivor count.
template <int S2, class Sink>
__device__ __forceinline__ int prepass3_more(const Args &a, Park3 *sv, int m, Sink &sink)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int m2 = 0;
    for (int r0 = 0; r0 < m; r0 += 32) {
        const bool valid = r0 + lane < m;
        Park3 p;
        p.o = 0u;
        p.x = p.y = 0.f;
        p.it = 0u;
        if (valid)
            p = sv[r0 + lane];
        bool surv = false;
        if (valid) {
            float cr, ci, w;
            voxel_c(a, p.o, cr, ci, w);
            float x = p.x, y = p.y, x2 = __fmul_rn(x, x), y2 = __fmul_rn(y, y);
            float inf_ = 0.0f;
#pragma unroll
            for (int k = 1; k <= S2; ++k) {
                MANDEL_STEP(x, y, x2, y2, cr, ci);
                inf_ = __fadd_rn(inf_, __fadd_rn(x2, y2) <= 4.0f ? 1.0f : 0.0f);
            }
            const int in_ = (int)inf_;
            if (in_ < S2) {
                sink(p.o, (int)p.it + in_ + 1);
            } else {
                surv = true;
                p.x = x;
                p.y = y;
                p.it += (unsigned)S2;
            }
        }
        const unsigned sm = __ballot_sync(FULL, surv); // every lane has read its record
        if (surv)
            sv[m2 + __popc(sm & lt)] = p;
        m2 += __popc(sm);
    }
    __syncwarp();
    return m2;
}

template <class Map, class Sink>
__device__ __forceinline__ void refill3_packed(const Args &a, unsigned long long total64, unsigned long long *cursor,
                                               const Map &map, Sink &sink, Park3 *q, Park3 *sv)
{
    const uint32_t total = (uint32_t)total64; // < n^3 <= 2^30
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t min_active = 8u * (uint32_t)c3_sms;
    uint32_t active = total / (64u * 8u);
    active = active < min_active ? min_active : active;
    active = active > nwarps ? nwarps : active;
    const uint32_t wrank = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    if (wrank >= active)
        return;
    uint32_t grab = total / (4u * active);
    grab = grab < 8u ? 8u : (grab > (uint32_t)PCH ? (uint32_t)PCH : grab);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned md = (unsigned)a.maxdwell;
    const bool use_pre = a.maxdwell > PPRE;
    bool exhausted = false;
    int qn = 0;
    uint32_t sv_pos = 0, sv_end = 0, pos = 0, end = 0;
    bool has0 = false, has1 = false, fin0 = false, fin1 = false;
    uint32_t o0 = 0, o1 = 0;
    unsigned it0 = 0, it1 = 0, sit0 = 0, sit1 = 0;
    float sx0 = 0.f, sy0 = 0.f, sx1 = 0.f, sy1 = 0.f;
    f2_t X = 0, Y = 0, X2 = 0, Y2 = 0, CR = 0, CI = 0;
    while (true) {
        const unsigned f0 = __ballot_sync(FULL, fin0), f1 = __ballot_sync(FULL, fin1);
        if (f0 | f1) {
            const int n0 = __popc(f0);
            if (fin0) {
                Park3 &e = q[qn + __popc(f0 & lt)];
                e.o = o0;
                e.x = sx0;
                e.y = sy0;
                e.it = sit0;
                has0 = false;
                fin0 = false;
            }
            if (fin1) {
                Park3 &e = q[qn + n0 + __popc(f1 & lt)];
                e.o = o1;
                e.x = sx1;
                e.y = sy1;
                e.it = sit1;
                has1 = false;
                fin1 = false;
            }
            qn += n0 + __popc(f1);
            __syncwarp();
            if (qn >= 64) {
                qn -= 64;
                replay3_2(a, q + qn, 64, md, sink);
            }
        }
        unsigned need0 = __ballot_sync(FULL, !has0), need1 = __ballot_sync(FULL, !has1);
        while ((need0 | need1) && !exhausted) {
            if (use_pre && sv_pos >= sv_end) { // prepass a fresh grab
                unsigned long long b = 0;
                if (lane == 0)
                    b = atomicAdd(cursor, (unsigned long long)grab);
                b = __shfl_sync(FULL, b, 0);
                if (b >= total) {
                    exhausted = true;
                    break;
                }
                const uint32_t e = (uint32_t)min(b + (unsigned long long)grab, (unsigned long long)total);
                sv_pos = 0;
                sv_end = (uint32_t)prepass3(a, (uint32_t)b, e, map, sink, sv);
                if constexpr (MANDEL3D_PRE2 > 0) {
                    if (a.maxdwell > PPRE + MANDEL3D_PRE2 && sv_end > 0)
                        sv_end = (uint32_t)prepass3_more<MANDEL3D_PRE2>(a, sv, (int)sv_end, sink);
                }
                continue;
            }
            // slots from the survivor buffer, or (no prepass) straight from the cursor
            const unsigned c0 = __popc(need0);
            const unsigned cnt = c0 + __popc(need1);
            unsigned take;
            uint32_t base;
            if (use_pre) {
                const unsigned avail = sv_end - sv_pos;
                take = avail < cnt ? avail : cnt;
                base = sv_pos;
            } else {
                if (pos >= end) {
                    unsigned long long b = 0;
                    if (lane == 0)
                        b = atomicAdd(cursor, (unsigned long long)grab);
                    b = __shfl_sync(FULL, b, 0);
                    if (b >= total) {
                        exhausted = true;
                        break;
                    }
                    pos = (uint32_t)b;
                    end = (uint32_t)min(b + (unsigned long long)grab, (unsigned long long)total);
                }
                const unsigned avail = end - pos;
                take = avail < cnt ? avail : cnt;
                base = pos;
            }
            const unsigned r0 = __popc(need0 & lt), r1 = c0 + __popc(need1 & lt);
            float cr0, ci0, cr1, ci1, xa0, xa1, ya0, ya1, qa0, qa1, wa0, wa1;
            f2_unpack(CR, cr0, cr1);
            f2_unpack(CI, ci0, ci1);
            f2_unpack(X, xa0, xa1);
            f2_unpack(Y, ya0, ya1);
            f2_unpack(X2, qa0, qa1);
            f2_unpack(Y2, wa0, wa1);
            bool new0 = false, new1 = false;
            for (int sl = 0; sl < 2; ++sl) {
                const bool want = sl == 0 ? (!has0 && r0 < take) : (!has1 && r1 < take);
                if (!want)
                    continue;
                const unsigned rk = sl == 0 ? r0 : r1;
                uint32_t o;
                float x, y;
                unsigned itv;
                float cr, ci, w;
                bool ok = true;
                if (use_pre) {
                    const Park3 pnt = sv[base + rk];
                    o = pnt.o;
                    voxel_c(a, o, cr, ci, w);
                    x = pnt.x;
                    y = pnt.y;
                    itv = pnt.it;
                } else {
                    o = map(base + rk);
                    voxel_c(a, o, cr, ci, w);
                    x = w;
                    y = 0.0f;
                    itv = 0;
                    if (!(__fadd_rn(__fmul_rn(cr, cr), __fmul_rn(ci, ci)) <= 3.9f)) {
                        sink(o, dwell3_per_step(cr, ci, w, a.maxdwell));
                        ok = false;
                    }
                }
                if (!ok)
                    continue;
                if (sl == 0) {
                    o0 = o; cr0 = cr; ci0 = ci; xa0 = x; ya0 = y;
                    qa0 = __fmul_rn(x, x); wa0 = __fmul_rn(y, y); it0 = itv; has0 = true; new0 = true;
                } else {
                    o1 = o; cr1 = cr; ci1 = ci; xa1 = x; ya1 = y;
                    qa1 = __fmul_rn(x, x); wa1 = __fmul_rn(y, y); it1 = itv; has1 = true; new1 = true;
                }
            }
            if (new0 | new1) {
                CR = f2_pack(cr0, cr1);
                CI = f2_pack(ci0, ci1);
                X = f2_pack(xa0, xa1);
                Y = f2_pack(ya0, ya1);
                X2 = f2_pack(qa0, qa1);
                Y2 = f2_pack(wa0, wa1);
            }
            if (use_pre)
                sv_pos += take;
            else
                pos += take;
            __syncwarp();
            need0 = __ballot_sync(FULL, !has0);
            need1 = __ballot_sync(FULL, !has1);
        }
        const unsigned a0m = __ballot_sync(FULL, has0), a1m = __ballot_sync(FULL, has1);
        if (!(a0m | a1m))
            break;
        const int thresh = exhausted ? 64 : PT;
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
            for (int k = 0; k < PK; ++k)
                MANDEL_STEP2(X, Y, X2, Y2, CR, CI);
            it0 += PK;
            it1 += PK;
            float m0, m1;
            f2_unpack(f2_add(X2, Y2), m0, m1);
            fin0 = live0 && (fin0 || !(m0 <= 4.0f) || it0 >= md);
            fin1 = live1 && (fin1 || !(m1 <= 4.0f) || it1 >= md);
            const unsigned g0 = __ballot_sync(FULL, fin0), g1 = __ballot_sync(FULL, fin1);
            if ((g0 == a0m && g1 == a1m) || __popc(g0) + __popc(g1) >= thresh)
                break;
        }
    }
    while (qn > 0) {
        const int c = qn < 64 ? qn : 64;
        qn -= c;
        replay3_2(a, q + qn, c, md, sink);
    }
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
__device__ __forceinline__ int plane_val(uint32_t i, int d) { return (int)(i / 2u + 1u) * d - 1 + (int)(i & 1u); }
__device__ __forceinline__ int off_val(const Args &a, uint32_t j)
{
    const uint32_t q = fdiv(j, a.fm);
    return (int)q * a.d + 1 + (int)(j - q * a.fm.d);
}
__device__ __forceinline__ void new_surface_voxel(const Args &a, uint32_t t, int &x, int &y, int &z)
{
    const uint32_t A2 = a.fa2.d, MA = a.fMa.d;
    const uint32_t Mv = a.fM.d;
    const uint32_t blk0 = Mv * A2; // x on a plane, y and z any interior value
    if (t < blk0) {
        const uint32_t i = fdiv(t, a.fa2), q = t - i * A2, qy = fdiv(q, a.fa);
        x = plane_val(i, a.d);
        y = 1 + (int)qy;
        z = 1 + (int)(q - qy * a.fa.d);
        return;
    }
    t -= blk0;
    const uint32_t blk1 = a.fm.d ? (uint32_t)(a.fNM.d / Mv) * MA : 0u; // N M a: x off, y on, z any
    if (t < blk1) {
        const uint32_t j = fdiv(t, a.fMa), q = t - j * MA, qy = fdiv(q, a.fa);
        x = off_val(a, j);
        y = plane_val(qy, a.d);
        z = 1 + (int)(q - qy * a.fa.d);
        return;
    }
    t -= blk1; // x, y off, z on a plane
    const uint32_t j = fdiv(t, a.fNM), q = t - j * a.fNM.d, qy = fdiv(q, a.fM);
    x = off_val(a, j);
    y = off_val(a, qy);
    z = plane_val(q - qy * Mv, a.d);
}

template <bool STATS>
__global__ void __launch_bounds__(256) k3_surface(Args a)
{
    __shared__ unsigned long long s_sum[8];
    // level 0: the whole surface of every region; level l > 0: the new plane voxels of every
    // region subdivided at level l-1 (its first child's corner is the parent's corner)
    const bool reuse = a.level > 0;
    const uint32_t units = reuse ? *((volatile uint32_t *)&a.hdr->n_subdiv[a.level - 1]) : level_count(a);
    const uint32_t total = a.fS.d * units;
    const uint32_t rrr = (uint32_t)(a.r * a.r * a.r);
    unsigned long long it = 0, px = 0;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const uint32_t p = fdiv(t, a.fS);
        int x0, y0, z0, x, y, z;
        unomega(a, a.olt_in[reuse ? p * rrr : p], x0, y0, z0);
        if (reuse)
            new_surface_voxel(a, t - p * a.fS.d, x, y, z);
        else
            surface_voxel(a, t - p * a.fS.d, x, y, z);
        x += x0;
        y += y0;
        z += z0;
        const int v = dwell3(vc(a.ax.x0, a.ax.dx, x), vc(a.ax.y0, a.ax.dy, y), vc(a.ax.z0, a.ax.dz, z), a.maxdwell);
        store_surface(a, x, y, z, v);
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
        for (uint32_t s = threadIdx.x; s < (uint32_t)S; s += blockDim.x) {
            int x, y, z;
            surface_voxel(a, s, x, y, z);
            // the slices' x-columns (x = 0 or d-1 off the z-faces) from the transposed planes
            const bool col = a.colT && s >= 2u * a.fdd.d && (x == 0 || x == a.d - 1);
            const int v = __ldcg(col ? a.colT + colT_idx(a, x0 + x, y0 + y, z0 + z)
                                     : a.out + vidx(a, x0 + x, y0 + y, z0 + z));
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

// Warp per region (small cubes: the block-per-region loop above spends most of a round in
// its two block barriers): the same reduction and decision, 8 regions per block in flight.
__global__ void __launch_bounds__(256) k3_classify_warp(Args a)
{
    const uint32_t count = level_count(a);
    const long long S = surface_count(a.d);
    const int rrr = a.r * a.r * a.r, h = a.d / a.r;
    const int lane = threadIdx.x & 31;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t ri = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ri < count; ri += warps) {
        const uint32_t off = a.olt_in[ri];
        int x0, y0, z0;
        unomega(a, off, x0, y0, z0);
        int lo = INT_MAX, hi = INT_MIN;
        for (uint32_t s = lane; s < (uint32_t)S; s += 32) {
            int x, y, z;
            surface_voxel(a, s, x, y, z);
            const bool col = a.colT && s >= 2u * a.fdd.d && (x == 0 || x == a.d - 1);
            const int v = __ldcg(col ? a.colT + colT_idx(a, x0 + x, y0 + y, z0 + z)
                                     : a.out + vidx(a, x0 + x, y0 + y, z0 + z));
            lo = min(lo, v);
            hi = max(hi, v);
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        uint32_t base = UINT_MAX;
        if (lane == 0) {
            if (lo == hi) {
                const uint32_t e = atomicAdd(&a.hdr->n_fill[a.level], 1u);
                a.fill[e] = make_uint2(off, (uint32_t)lo);
            } else if (a.subdivide) {
                base = atomicAdd(&a.hdr->n_subdiv[a.level], 1u);
            } else {
                a.leaf[atomicAdd(&a.hdr->n_leaf, 1u)] = off;
            }
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base != UINT_MAX)
            for (int c = lane; c < rrr; c += 32) {
                const int cx = c % a.r, cy = (c / a.r) % a.r, cz = c / (a.r * a.r);
                a.olt_out[(size_t)base * rrr + c] = omega(a, x0 + cx * h, y0 + cy * h, z0 + cz * h);
            }
    }
}

// Uniform cubes: flat over all voxels of the level's filled regions; int4 stores along x
// when d % 4 == 0 (rows 16-byte aligned: the volume base is 256-byte aligned and n % 4 == 0).
template <bool VEC>
__global__ void __launch_bounds__(256) k3_fill(Args a)
{
    const uint32_t count = *((volatile uint32_t *)&a.hdr->n_fill[a.level]);
    const int d = a.d;
    const uint32_t total = count << a.log_fill_per; // units: int4 (VEC) or int
    const uint32_t rmask = (1u << a.log_fill_row) - 1u, dmask = (uint32_t)d - 1u;
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < total; u += gridDim.x * blockDim.x) {
        const uint32_t e = u >> a.log_fill_per;
        const uint32_t rem = u - (e << a.log_fill_per);
        const uint2 f = a.fill[e];
        int x0, y0, z0;
        unomega(a, f.x, x0, y0, z0);
        const int ux = (int)(rem & rmask), y = (int)((rem >> a.log_fill_row) & dmask),
                  z = (int)(rem >> (a.log_fill_row + a.log_d));
        const int v = (int)f.y;
        if (VEC)
            __stcs(reinterpret_cast<int4 *>(a.out + vidx(a, x0 + 4 * ux, y0 + y, z0 + z)), make_int4(v, v, v, v));
        else
            a.out[vidx(a, x0 + ux, y0 + y, z0 + z)] = v;
    }
}

// Flat index -> voxel maps of the surface and leaf kernels, for the lane-refill engine.
struct SurfMap {
    Args a;
    bool reuse;
    __device__ __forceinline__ uint32_t operator()(unsigned long long tt) const
    {
        const uint32_t t = (uint32_t)tt, p = fdiv(t, a.fS);
        int x0, y0, z0, x, y, z;
        unomega(a, a.olt_in[reuse ? p * (uint32_t)(a.r * a.r * a.r) : p], x0, y0, z0);
        if (reuse)
            new_surface_voxel(a, t - p * a.fS.d, x, y, z);
        else
            surface_voxel(a, t - p * a.fS.d, x, y, z);
        return omega(a, x0 + x, y0 + y, z0 + z);
    }
};
struct LeafMap3 {
    Args a;
    __device__ __forceinline__ uint32_t operator()(unsigned long long tt) const
    {
        const uint32_t t = (uint32_t)tt, li = fdiv(t, a.fI), loc = t - li * a.fI.d;
        const uint32_t q = fdiv(loc, a.fm), lz = fdiv(q, a.fm);
        int x0, y0, z0;
        unomega(a, a.leaf[li], x0, y0, z0);
        return omega(a, x0 + 1 + (int)(loc - q * a.fm.d), y0 + 1 + (int)(q - lz * a.fm.d), z0 + 1 + (int)lz);
    }
};

#ifndef MANDEL3D_CLASSIFY_WARP_D // warp per region for cube sides up to this
#define MANDEL3D_CLASSIFY_WARP_D 32
#endif
#ifndef MANDEL3D_SURF_PACK
#define MANDEL3D_SURF_PACK 1 // surfaces on the packed FFMA2 engine (0: the scalar refill3)
#endif
template <bool STATS>
__global__ void __launch_bounds__(RTPB, MANDEL3D_SURF_PACK ? PMINB : RMINB) k3_surface_rf(Args a)
{
    __shared__ unsigned long long s_sum[RTPB / 32];
    const bool reuse = a.level > 0;
    SurfMap map{a, reuse};
    const uint32_t units = reuse ? *((volatile uint32_t *)&a.hdr->n_subdiv[a.level - 1]) : level_count(a);
    Sink3<STATS> sink{&a, 0ull, 0ull};
#if MANDEL3D_SURF_PACK
    __shared__ Park3 s_q[RTPB / 32][128];
    __shared__ Park3 s_sv[RTPB / 32][PCH];
    refill3_packed(a, (unsigned long long)a.fS.d * units, &a.hdr->cursor[a.level], map, sink, s_q[threadIdx.x >> 5],
                   s_sv[threadIdx.x >> 5]);
#else
    __shared__ Park3 s_q[RTPB / 32][64];
    refill3(a, (unsigned long long)a.fS.d * units, &a.hdr->cursor[a.level], map, sink, s_q[threadIdx.x >> 5]);
#endif
    if (STATS) {
        const unsigned long long it = block_sum<RTPB>(sink.iters, s_sum);
        if (threadIdx.x == 0 && it)
            atomicAdd(&a.hdr->border_iters[a.level], it);
        const unsigned long long px = block_sum<RTPB>(sink.px, s_sum);
        if (threadIdx.x == 0 && px)
            atomicAdd(&a.hdr->border_px[a.level], px);
    }
}

#ifndef MANDEL3D_LEAF_PACK
#define MANDEL3D_LEAF_PACK 1 // leaves on the packed FFMA2 engine (0: the scalar refill3)
#endif
template <bool STATS>
__global__ void __launch_bounds__(RTPB, MANDEL3D_LEAF_PACK ? PMINB : RMINB) k3_leaf_rf(Args a)
{
    __shared__ unsigned long long s_sum[RTPB / 32];
    LeafMap3 map{a};
    Sink3<STATS, false> sink{&a, 0ull, 0ull};
#if MANDEL3D_LEAF_PACK
    __shared__ Park3 s_q[RTPB / 32][128];
    __shared__ Park3 s_sv[RTPB / 32][PCH];
    if (a.fI.d > 0)
        refill3_packed(a, (unsigned long long)a.fI.d * *((volatile uint32_t *)&a.hdr->n_leaf), &a.hdr->cursor[MAXL],
                       map, sink, s_q[threadIdx.x >> 5], s_sv[threadIdx.x >> 5]);
#else
    __shared__ Park3 s_q[RTPB / 32][64];
    if (a.fI.d > 0)
        refill3(a, (unsigned long long)a.fI.d * *((volatile uint32_t *)&a.hdr->n_leaf), &a.hdr->cursor[MAXL], map,
                sink, s_q[threadIdx.x >> 5]);
#endif
    if (STATS) {
        const unsigned long long it = block_sum<RTPB>(sink.iters, s_sum);
        if (threadIdx.x == 0 && it)
            atomicAdd(&a.hdr->leaf_iters, it);
        const unsigned long long px = block_sum<RTPB>(sink.px, s_sum);
        if (threadIdx.x == 0 && px)
            atomicAdd(&a.hdr->leaf_px, px);
    }
}

template <bool STATS>
__global__ void __launch_bounds__(256) k3_leaf(Args a)
{
    __shared__ unsigned long long s_sum[8];
    const uint32_t total = a.fI.d * *((volatile uint32_t *)&a.hdr->n_leaf);
    const LeafMap3 map{a};
    unsigned long long it = 0, px = 0;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        int x, y, z;
        unomega(a, map(t), x, y, z);
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
    size_t hdr, olt[2], fill, leaf, colT, colT_bytes, total;
    int log_u;
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
    int64_t u = n / g; // leaf side
    for (int l = 1; l < lay.L; ++l)
        u /= r;
    lay.log_u = lg2(u);
    lay.colT = o;
    lay.colT_bytes = u >= 8 ? (size_t)(2 * (n / u)) * (size_t)n * (size_t)n * 4 : 0;
    o = a256(o + lay.colT_bytes);
    lay.total = o;
    return true;
}

FastDiv nz_div(uint32_t d) // divisor 0 marks an empty index space (the map is never evaluated)
{
    if (d == 0) {
        FastDiv f{0u, 0u, 0u, 0u};
        return f;
    }
    return make_fastdiv(d);
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

// per device: the fill side stream and its fork/join events (mandel3d_shutdown frees them)
cudaStream_t g_side[16] = {};
cudaEvent_t g_fork[16] = {}, g_join[16] = {};

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
    if (!valid_region(reg) || maxdwell < 1 || !d_out || !d_ws || (flags & ~(MANDEL3D_FLAG_STATS | MANDEL3D_FLAG_FLAT)) ||
        !make_layout(n, g, r, B, lay) || ((uintptr_t)d_ws % 256) != 0 || ((uintptr_t)d_out % 16) != 0)
        return 1;
    if (ws_bytes < lay.total)
        return 2;
    const bool stats = (flags & MANDEL3D_FLAG_STATS) != 0;
    const bool flat = (flags & MANDEL3D_FLAG_FLAT) != 0;
    cudaStream_t s = (cudaStream_t)stream;
    // fills (HBM-bound, terminal: no later kernel reads a filled cube's interior) run on a side
    // stream forked after each level's classification and joined at the end (as the 2-D path)
    cudaStream_t *side = g_side;
    cudaEvent_t *ev_fork = g_fork, *ev_join = g_join;
    int cur = 0;
    CK3(cudaGetDevice(&cur));
    if (cur >= 16)
        return 1;
    if (!side[cur]) {
        CK3(cudaStreamCreateWithFlags(&side[cur], cudaStreamNonBlocking));
        CK3(cudaEventCreateWithFlags(&ev_fork[cur], cudaEventDisableTiming));
        CK3(cudaEventCreateWithFlags(&ev_join[cur], cudaEventDisableTiming));
    }
    cudaStream_t sf = side[cur];
    // the side stream must not run ahead of work the caller queued before this call
    CK3(cudaEventRecord(ev_fork[cur], s));
    CK3(cudaStreamWaitEvent(sf, ev_fork[cur], 0));
    {
        static int sms_dev = -1; // c3_sms of the current device (the engine's active-warp floor)
        int dev = 0, sms = 0;
        CK3(cudaGetDevice(&dev));
        if (dev != sms_dev) {
            CK3(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            CK3(cudaMemcpyToSymbol(c3_sms, &sms, sizeof sms));
            sms_dev = dev;
        }
    }
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
    if (lay.colT_bytes) {
        a.colT = (int *)(ws + lay.colT);
        a.log_u = lay.log_u;
    }
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
        {
            const uint32_t A = (uint32_t)(r * d - 2), M = (uint32_t)(2 * (r - 1)), N = (uint32_t)(r * (d - 2));
            const uint32_t m = (uint32_t)(d - 2);
            a.fS = make_fastdiv((uint32_t)(l == 0 ? surface_count(d) : new_surface_count(d, r)));
            a.fdd = make_fastdiv((uint32_t)(d * d));
            a.fd = make_fastdiv((uint32_t)d);
            a.fring = make_fastdiv((uint32_t)(4 * d - 4));
            a.fa2 = make_fastdiv(A * A);
            a.fa = make_fastdiv(A);
            a.fMa = make_fastdiv(M * A);
            a.fNM = nz_div(N * M);
            a.fM = make_fastdiv(M);
            a.fm = nz_div(m);
            a.fI = nz_div(m * m * m);
            const bool v4 = d % 4 == 0;
            a.log_d = lg2(d);
            a.log_fill_row = lg2(v4 ? d / 4 : d);
            a.log_fill_per = a.log_fill_row + 2 * a.log_d;
        }
        const size_t cap = lay.cap[l];
        const size_t sblocks = (l == 0 ? cap * (size_t)surface_count(d)
                                       : cap / ((size_t)r * r * r) * (size_t)new_surface_count(d, r)) / 256 + 1;
        if (flat && stats)
            k3_surface<true><<<resident(k3_surface<true>, 256, sblocks), 256, 0, s>>>(a);
        else if (flat)
            k3_surface<false><<<resident(k3_surface<false>, 256, sblocks), 256, 0, s>>>(a);
        else if (stats)
            k3_surface_rf<true><<<resident(k3_surface_rf<true>, RTPB, sblocks), RTPB, 0, s>>>(a);
        else
            k3_surface_rf<false><<<resident(k3_surface_rf<false>, RTPB, sblocks), RTPB, 0, s>>>(a);
        CK3(cudaGetLastError());
        if (d <= MANDEL3D_CLASSIFY_WARP_D)
            k3_classify_warp<<<resident(k3_classify_warp, 256, (cap + 7) / 8), 256, 0, s>>>(a);
        else
            k3_classify<<<resident(k3_classify, 256, cap), 256, 0, s>>>(a);
        CK3(cudaGetLastError());
        const bool vec = d % 4 == 0;
        const size_t fblocks = (cap * (size_t)d * d * d / (vec ? 4 : 1) + 255) / 256;
        CK3(cudaEventRecord(ev_fork[cur], s)); // fork: this level's fill waits for its classify
        CK3(cudaStreamWaitEvent(sf, ev_fork[cur], 0));
        if (vec)
            k3_fill<true><<<resident(k3_fill<true>, 256, fblocks), 256, 0, sf>>>(a);
        else
            k3_fill<false><<<resident(k3_fill<false>, 256, fblocks), 256, 0, sf>>>(a);
        CK3(cudaGetLastError());
        if (l + 1 < lay.L)
            d /= r;
    }
    const size_t lblocks = (lay.cap[lay.L - 1] * (size_t)(d > 2 ? d - 2 : 0) * (d > 2 ? d - 2 : 0) *
                                (d > 2 ? d - 2 : 0) + 255) / 256;
    if (lblocks > 0) {
        if (flat && stats)
            k3_leaf<true><<<resident(k3_leaf<true>, 256, lblocks), 256, 0, s>>>(a);
        else if (flat)
            k3_leaf<false><<<resident(k3_leaf<false>, 256, lblocks), 256, 0, s>>>(a);
        else if (stats)
            k3_leaf_rf<true><<<resident(k3_leaf_rf<true>, RTPB, lblocks), RTPB, 0, s>>>(a);
        else
            k3_leaf_rf<false><<<resident(k3_leaf_rf<false>, RTPB, lblocks), RTPB, 0, s>>>(a);
        CK3(cudaGetLastError());
    }
    CK3(cudaEventRecord(ev_join[cur], sf)); // join the fills
    CK3(cudaStreamWaitEvent(s, ev_join[cur], 0));
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

void mandel3d_shutdown(void)
{
    int prev = 0;
    cudaGetDevice(&prev);
    for (int d = 0; d < 16; ++d) {
        if (!g_side[d])
            continue;
        cudaSetDevice(d);
        cudaStreamSynchronize(g_side[d]);
        cudaStreamDestroy(g_side[d]);
        cudaEventDestroy(g_fork[d]);
        cudaEventDestroy(g_join[d]);
        g_side[d] = nullptr;
        g_fork[d] = g_join[d] = nullptr;
    }
    cudaSetDevice(prev);
}

} // extern "C"
