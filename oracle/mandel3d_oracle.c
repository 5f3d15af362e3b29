/*
 * mandel3d_oracle.c -- CPU ORACLE for the 3-D (k = 3) ASK path.  TEST INFRASTRUCTURE ONLY.
 *
 * Same status as mandel_oracle.c: only tests/ (and smoke()) load it; the product never links,
 * imports or executes it and shares no code with it.  Plain, slow, single-threaded C, built
 * with gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math (one IEEE binary32 RN operation per
 * written operation, no FMA contraction).
 *
 * The paper's Sec. 6.2 ("Subdivisions at Higher Dimensions") extends ASK to a
 * k-orthotope domain: g^k initial regions, each subdividing into r^k sub-orthotopes
 * (P:555), with the offsets-lookup table holding one scalar per region through a
 * space-filling curve.  The paper gives no 3-D workload; DESIGN.md readings
 * R15-R17 fix this one:
 *   R15  domain: the 3-D slice (c_re, c_im, w) of the quadratic family's parameter space,
 *        z_{i+1} = z_i^2 + c from z_0 = w + 0i (w = 0 is the Mandelbrot set of the 2-D path);
 *        dwell = first i >= 1 with |z_i|^2 > 4, else maxdwell, in the operation order of
 *        reading R4;
 *   R16  voxel (x, y, z) samples its centre, each axis exactly like reading R3;
 *   R17  a region's "border" is its surface: the d^3 - (d-2)^3 voxels with at least one
 *        coordinate on the cube's boundary (the k = 3 analogue of the 4d-4 ring, R7); the
 *        decision rule is unchanged (uniform -> fill, else subdivide iff d/r >= B, else leaf).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double re_min, re_max, im_min, im_max, w_min, w_max;
} oracle3_region;

typedef struct {
    int64_t regions_in, filled, subdivided, leaves;
    int64_t border_px, border_iters; /* surface voxels evaluated, sum of their dwells        */
    int64_t leaf_px, leaf_iters;     /* interior voxels of leaves, sum of their dwells       */
} oracle3_level_stats;

/* Dwell with z_0 = w (R15). */
int32_t oracle3_dwell(float cr, float ci, float w, int32_t maxdwell)
{
    float x = w, y = 0.0f;
    for (int32_t i = 1; i <= maxdwell; ++i) {
        float x2 = x * x;
        float y2 = y * y;
        float xy = x * y;
        x = (x2 - y2) + cr;
        y = (xy + xy) + ci;
        float mag = x * x + y * y;
        if (mag > 4.0f)
            return i;
    }
    return maxdwell;
}

/* Voxel (x, y, z) -> (cr, ci, w) at the voxel centre (R16): per axis
 *   v = (float)lo + ((float)k + 0.5f) * (float)((hi - lo) / n), the division in double. */
void oracle3_voxel_c(oracle3_region reg, int64_t n, int64_t x, int64_t y, int64_t z, float *cr, float *ci,
                     float *w)
{
    float x0 = (float)reg.re_min, dx = (float)((reg.re_max - reg.re_min) / (double)n);
    float y0 = (float)reg.im_min, dy = (float)((reg.im_max - reg.im_min) / (double)n);
    float z0 = (float)reg.w_min, dz = (float)((reg.w_max - reg.w_min) / (double)n);
    float fx = (float)x + 0.5f, fy = (float)y + 0.5f, fz = (float)z + 0.5f;
    *cr = x0 + fx * dx;
    *ci = y0 + fy * dy;
    *w = z0 + fz * dz;
}

static int32_t voxel_dwell(oracle3_region reg, int64_t n, int32_t maxdwell, int64_t x, int64_t y, int64_t z)
{
    float cr, ci, w;
    oracle3_voxel_c(reg, n, x, y, z, &cr, &ci, &w);
    return oracle3_dwell(cr, ci, w, maxdwell);
}

/* Exhaustive volume, z-slices [z0, z0 + nz): out[((z - z0) * n + y) * n + x]. */
void oracle3_exhaustive_slices(oracle3_region reg, int64_t n, int32_t maxdwell, int64_t z0, int64_t nz,
                               int32_t *out)
{
    for (int64_t z = z0; z < z0 + nz; ++z)
        for (int64_t y = 0; y < n; ++y)
            for (int64_t x = 0; x < n; ++x)
                out[((z - z0) * n + y) * n + x] = voxel_dwell(reg, n, maxdwell, x, y, z);
}

/* --------------------------------------------------------------------------------------
 * Recursive 3-D Mariani-Silver / ASK (P:216 with the k = 3 orthotopes of P:553-555): for each
 * of the g^3 level-0 cubes in canonical order (cz, cy, cx), examine the surface; uniform ->
 * fill the cube; else if d / r >= B -> the r^3 sub-cubes in canonical order; else every voxel.
 * ------------------------------------------------------------------------------------ */
typedef struct {
    oracle3_region reg;
    int64_t n;
    int32_t maxdwell;
    int r, B;
    const int32_t *lookup; /* NULL: compute dwells; else read them from this n^3 volume      */
    int32_t *out;          /* voxel (x, y, z) at out[((z-oz) * wy + (y-oy)) * wx + (x-ox)]   */
    int64_t ox, oy, oz, wx, wy;
    oracle3_level_stats *stats;
    int max_levels;
    int error;
} ask3_ctx;

static int32_t ctx3_dwell(ask3_ctx *c, int64_t x, int64_t y, int64_t z)
{
    if (c->lookup)
        return c->lookup[(z * c->n + y) * c->n + x];
    return voxel_dwell(c->reg, c->n, c->maxdwell, x, y, z);
}

static int32_t *ctx3_at(ask3_ctx *c, int64_t x, int64_t y, int64_t z)
{
    return &c->out[((z - c->oz) * c->wy + (y - c->oy)) * c->wx + (x - c->ox)];
}

static void ask3_region(ask3_ctx *c, int64_t x0, int64_t y0, int64_t z0, int64_t d, int level)
{
    if (level >= c->max_levels) {
        c->error = 1;
        return;
    }
    oracle3_level_stats *st = c->stats ? &c->stats[level] : NULL;
    if (st)
        st->regions_in++;
    int uniform = 1, first = 1;
    int32_t v = 0;
    for (int64_t z = z0; z < z0 + d; ++z)
        for (int64_t y = y0; y < y0 + d; ++y)
            for (int64_t x = x0; x < x0 + d; ++x) {
                int on_surface = (x == x0 || x == x0 + d - 1 || y == y0 || y == y0 + d - 1 || z == z0 ||
                                  z == z0 + d - 1);
                if (!on_surface)
                    continue;
                int32_t u = ctx3_dwell(c, x, y, z);
                if (st) {
                    st->border_px++;
                    st->border_iters += u;
                }
                if (first) {
                    v = u;
                    first = 0;
                } else if (u != v) {
                    uniform = 0;
                }
            }
    if (uniform) {
        for (int64_t z = z0; z < z0 + d; ++z)
            for (int64_t y = y0; y < y0 + d; ++y)
                for (int64_t x = x0; x < x0 + d; ++x)
                    *ctx3_at(c, x, y, z) = v;
        if (st)
            st->filled++;
        return;
    }
    if (d / c->r >= c->B) {
        int64_t s = d / c->r;
        if (st)
            st->subdivided++;
        for (int cz = 0; cz < c->r; ++cz)
            for (int cy = 0; cy < c->r; ++cy)
                for (int cx = 0; cx < c->r; ++cx)
                    ask3_region(c, x0 + cx * s, y0 + cy * s, z0 + cz * s, s, level + 1);
        return;
    }
    for (int64_t z = z0; z < z0 + d; ++z)
        for (int64_t y = y0; y < y0 + d; ++y)
            for (int64_t x = x0; x < x0 + d; ++x) {
                int32_t u = ctx3_dwell(c, x, y, z);
                *ctx3_at(c, x, y, z) = u;
                int interior = !(x == x0 || x == x0 + d - 1 || y == y0 || y == y0 + d - 1 || z == z0 ||
                                 z == z0 + d - 1);
                if (st && interior) {
                    st->leaf_px++;
                    st->leaf_iters += u;
                }
            }
    if (st)
        st->leaves++;
}

/* tiles: canonical level-0 ids k = (gz * g + gy) * g + gx (NULL: all g^3 in that order).
 * Returns 0 on success, 1 on invalid arguments, 2 if more than max_levels were needed. */
static int run_ask3(ask3_ctx *c, int g, const int32_t *tiles, int64_t ntiles)
{
    int64_t n = c->n;
    if (n <= 0 || g <= 0 || c->r < 2 || c->B < 1 || n % g != 0 || (n / g) < c->B)
        return 1;
    int64_t d0 = n / g, G = (int64_t)g * g * g;
    if (c->stats)
        memset(c->stats, 0, sizeof(oracle3_level_stats) * (size_t)c->max_levels);
    int64_t count = tiles ? ntiles : G;
    for (int64_t t = 0; t < count; ++t) {
        int64_t k = tiles ? tiles[t] : t;
        if (k < 0 || k >= G)
            return 1;
        int64_t gx = k % g, gy = (k / g) % g, gz = k / ((int64_t)g * g);
        ask3_region(c, gx * d0, gy * d0, gz * d0, d0, 0);
    }
    return c->error ? 2 : 0;
}

int oracle3_ask_window(oracle3_region reg, int64_t n, int32_t maxdwell, int g, int r, int B, const int32_t *tiles,
                       int64_t ntiles, int32_t *out, int64_t ox, int64_t oy, int64_t oz, int64_t wx, int64_t wy,
                       oracle3_level_stats *stats, int max_levels)
{
    ask3_ctx c;
    memset(&c, 0, sizeof c);
    c.reg = reg;
    c.n = n;
    c.maxdwell = maxdwell;
    c.r = r;
    c.B = B;
    c.out = out;
    c.ox = ox;
    c.oy = oy;
    c.oz = oz;
    c.wx = wx;
    c.wy = wy;
    c.stats = stats;
    c.max_levels = max_levels;
    if (maxdwell < 1)
        return 1;
    return run_ask3(&c, g, tiles, ntiles);
}

int oracle3_ask_by_lookup(const int32_t *E, int64_t n, int g, int r, int B, int32_t *out,
                          oracle3_level_stats *stats, int max_levels)
{
    ask3_ctx c;
    memset(&c, 0, sizeof c);
    c.n = n;
    c.r = r;
    c.B = B;
    c.lookup = E;
    c.out = out;
    c.wx = n;
    c.wy = n;
    c.stats = stats;
    c.max_levels = max_levels;
    return run_ask3(&c, g, NULL, 0);
}
