/*
 * mandel_oracle.c -- CPU ORACLE for the ASK Mandelbrot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  The product (paper_2206_02255_b200/) never links, imports or
 * executes it, and this file shares no code, header, table or constant with the CUDA path.
 *
 * Plain, slow, single-threaded, obviously-correct C.  Every function cites the passage of
 * /root/reference/PAPER.md (P:NNN = line NNN) it writes out.  Build flags (oracle/build.py):
 * gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math, so every float operation below is one
 * IEEE-754 binary32 operation rounded to nearest, in the order written (x86-64 SSE,
 * FLT_EVAL_METHOD == 0, no FMA contraction, no FTZ/DAZ).
 *
 * Precision and op order are DESIGN.md readings R2-R4 (the paper does not state them):
 * FP32 round-to-nearest, z_0 = 0, dwell = first i >= 1 with |z_i|^2 > 4, else maxdwell.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double re_min, re_max, im_min, im_max;
} oracle_region;

/* Per-level statistics of one ASK run (SPEC.md S:274-277 LevelStats, extended). */
typedef struct {
    int64_t regions_in;   /* regions examined at this level                        */
    int64_t filled;       /* uniform border -> filled with the border dwell         */
    int64_t subdivided;   /* non-uniform, d/r >= B -> r*r children at level+1        */
    int64_t leaves;       /* non-uniform, d/r <  B -> per-pixel dwell               */
    int64_t border_px;    /* border pixels evaluated (4d-4 per region)              */
    int64_t border_iters; /* sum of their dwells (= iterations executed)            */
    int64_t leaf_px;      /* interior pixels of leaves ((d-2)^2 per leaf)           */
    int64_t leaf_iters;   /* sum of their dwells                                    */
} oracle_level_stats;

/* One terminal region of the subdivision (for tiling / coverage tests). */
typedef struct {
    int32_t x, y, d, kind, value, level; /* kind 0 = filled (value = fill), 1 = leaf */
} oracle_region_rec;

/* --------------------------------------------------------------------------------------
 * Dwell (Sec. 7): z_{i+1} = z_i^2 + c, z_0 = 0; the dwell is the number of
 * iterations before |z| > 2 is detected, capped at maxdwell.  Written out in FP32 with
 * the operation order of DESIGN.md R4:  x2 = x*x, y2 = y*y, xy = x*y,
 * x = (x2 - y2) + cr, y = (xy + xy) + ci, escape iff x*x + y*y > 4 (strict).
 * ------------------------------------------------------------------------------------ */
int32_t oracle_dwell(float cr, float ci, int32_t maxdwell)
{
    float x = 0.0f, y = 0.0f;
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

/* Pixel (i, j) -> c at the pixel centre (R3):
 *   cr = (float)re_min + ((float)j + 0.5f) * (float)((re_max - re_min) / n)
 *   ci = (float)im_min + ((float)i + 0.5f) * (float)((im_max - im_min) / n)
 * Row i = 0 is the im_min side.  The width/n division is done once in double. */
void oracle_pixel_c(oracle_region reg, int64_t n, int64_t i, int64_t j, float *cr, float *ci)
{
    float x0 = (float)reg.re_min;
    float y0 = (float)reg.im_min;
    float dx = (float)((reg.re_max - reg.re_min) / (double)n);
    float dy = (float)((reg.im_max - reg.im_min) / (double)n);
    float tj = (float)j + 0.5f;
    float ti = (float)i + 0.5f;
    float pj = tj * dx;
    float pi_ = ti * dy;
    *cr = x0 + pj;
    *ci = y0 + pi_;
}

static int32_t pixel_dwell(oracle_region reg, int64_t n, int32_t maxdwell, int64_t i, int64_t j)
{
    float cr, ci;
    oracle_pixel_c(reg, n, i, j, &cr, &ci);
    return oracle_dwell(cr, ci, maxdwell);
}

/* Exhaustive approach Ex (P:111-117 eq:exhaustive-general): the dwell of every
 * pixel.  Computes rows [row0, row0 + rows) into out[(i - row0) * n + j]. */
void oracle_exhaustive_rows(oracle_region reg, int64_t n, int32_t maxdwell,
                            int64_t row0, int64_t rows, int32_t *out)
{
    for (int64_t i = row0; i < row0 + rows; ++i)
        for (int64_t j = 0; j < n; ++j)
            out[(i - row0) * n + j] = pixel_dwell(reg, n, maxdwell, i, j);
}

void oracle_exhaustive(oracle_region reg, int64_t n, int32_t maxdwell, int32_t *out)
{
    oracle_exhaustive_rows(reg, n, maxdwell, 0, n, out);
}

/* Sampled exhaustive: dwell of the listed pixels (ii[k], jj[k]). */
void oracle_dwell_pixels(oracle_region reg, int64_t n, int32_t maxdwell, const int64_t *ii,
                         const int64_t *jj, int64_t count, int32_t *out)
{
    for (int64_t k = 0; k < count; ++k)
        out[k] = pixel_dwell(reg, n, maxdwell, ii[k], jj[k]);
}

/* --------------------------------------------------------------------------------------
 * ASK / Mariani-Silver subdivision, written as the plain recursion (Sec. 4.2.1;
 * P:413, Sec. 7; ASK evaluates the same decisions level by level):
 *   region(x0, y0, d):
 *     compute the dwell of the 4d-4 border pixels             (query Q)
 *     if all equal v: write v to all d*d pixels               (terminal work T)
 *     elif d / r >= B: recurse into the r x r children         (subdivision S)
 *     else: dwell of every pixel of the region                 (last-level work L)
 * Stopping rule "subdivide iff d / r >= B" is DESIGN.md reading R5; filling at every level
 * (level 0 and the last level included) is reading R6.
 *
 * The dwell source is either the dwell function (oracle_ask) or a precomputed exhaustive
 * image (oracle_ask_by_lookup).
 * ------------------------------------------------------------------------------------ */
typedef struct {
    oracle_region reg;
    int64_t n;
    int32_t maxdwell;
    int r, B;
    const int32_t *lookup; /* NULL: compute dwells; else read them from this n x n image */
    int32_t *out;          /* pixel (x, y) is stored at out[(y - oy) * opitch + (x - ox)]  */
    int64_t ox, oy, opitch;
    oracle_level_stats *stats;
    int max_levels;
    oracle_region_rec *recs;
    int64_t rec_cap, rec_count;
    int error;
} ask_ctx;

static int32_t ctx_dwell(ask_ctx *c, int64_t x, int64_t y)
{
    /* x = column j, y = row i */
    if (c->lookup)
        return c->lookup[y * c->n + x];
    return pixel_dwell(c->reg, c->n, c->maxdwell, y, x);
}

static void add_rec(ask_ctx *c, int64_t x0, int64_t y0, int64_t d, int kind, int32_t v, int level)
{
    if (!c->recs)
        return;
    if (c->rec_count < c->rec_cap) {
        oracle_region_rec *q = &c->recs[c->rec_count];
        q->x = (int32_t)x0;
        q->y = (int32_t)y0;
        q->d = (int32_t)d;
        q->kind = kind;
        q->value = v;
        q->level = level;
    }
    c->rec_count++;
}

static void ask_region(ask_ctx *c, int64_t x0, int64_t y0, int64_t d, int level)
{
    oracle_level_stats *st = NULL;
    if (level >= c->max_levels) {
        c->error = 1;
        return;
    }
    if (c->stats)
        st = &c->stats[level];
    if (st)
        st->regions_in++;

    /* Border set: pixels of the region with x in {x0, x0+d-1} or y in {y0, y0+d-1}. */
    int uniform = 1;
    int32_t v = 0;
    int first = 1;
    for (int64_t y = y0; y < y0 + d; ++y) {
        for (int64_t x = x0; x < x0 + d; ++x) {
            int on_border = (x == x0 || x == x0 + d - 1 || y == y0 || y == y0 + d - 1);
            if (!on_border)
                continue;
            int32_t w = ctx_dwell(c, x, y);
            if (st) {
                st->border_px++;
                st->border_iters += w;
            }
            if (first) {
                v = w;
                first = 0;
            } else if (w != v) {
                uniform = 0;
            }
        }
    }

    if (uniform) {
        for (int64_t y = y0; y < y0 + d; ++y)
            for (int64_t x = x0; x < x0 + d; ++x)
                c->out[(y - c->oy) * c->opitch + (x - c->ox)] = v;
        if (st)
            st->filled++;
        add_rec(c, x0, y0, d, 0, v, level);
        return;
    }
    if (d / c->r >= c->B) {
        int64_t s = d / c->r;
        if (st)
            st->subdivided++;
        for (int cy = 0; cy < c->r; ++cy)
            for (int cx = 0; cx < c->r; ++cx)
                ask_region(c, x0 + cx * s, y0 + cy * s, s, level + 1);
        return;
    }
    /* Leaf: per-pixel dwell of every pixel of the region. */
    for (int64_t y = y0; y < y0 + d; ++y) {
        for (int64_t x = x0; x < x0 + d; ++x) {
            int32_t w = ctx_dwell(c, x, y);
            c->out[(y - c->oy) * c->opitch + (x - c->ox)] = w;
            int interior = !(x == x0 || x == x0 + d - 1 || y == y0 || y == y0 + d - 1);
            if (st && interior) {
                st->leaf_px++;
                st->leaf_iters += w;
            }
        }
    }
    if (st)
        st->leaves++;
    add_rec(c, x0, y0, d, 1, 0, level);
}

/* Runs the subdivision over the level-0 tiles listed in tiles[0..ntiles) (canonical index
 * k = gy * g + gx), or over all g*g tiles in canonical order when tiles == NULL.
 * Returns 0 on success, 1 on invalid arguments, 2 if more than max_levels levels were
 * needed, 3 if the region record buffer was too small (rec_count still set). */
static int run_ask(ask_ctx *c, int g, const int32_t *tiles, int64_t ntiles, int64_t *rec_count)
{
    int64_t n = c->n;
    if (n <= 0 || g <= 0 || c->r < 2 || c->B < 1 || n % g != 0 || (n / g) < c->B)
        return 1;
    int64_t d0 = n / g;
    if (c->stats)
        memset(c->stats, 0, sizeof(oracle_level_stats) * (size_t)c->max_levels);
    int64_t count = tiles ? ntiles : (int64_t)g * g;
    for (int64_t t = 0; t < count; ++t) {
        int64_t k = tiles ? tiles[t] : t;
        if (k < 0 || k >= (int64_t)g * g)
            return 1;
        int64_t gx = k % g, gy = k / g;
        ask_region(c, gx * d0, gy * d0, d0, 0);
    }
    if (rec_count)
        *rec_count = c->rec_count;
    if (c->error)
        return 2;
    if (c->recs && c->rec_count > c->rec_cap)
        return 3;
    return 0;
}

/* The output window: pixels are stored at out[(y - oy) * opitch + (x - ox)]; the caller
 * guarantees that every pixel of the listed tiles falls inside it. */
int oracle_ask_window(oracle_region reg, int64_t n, int32_t maxdwell, int g, int r, int B,
                      const int32_t *tiles, int64_t ntiles, int32_t *out, int64_t ox, int64_t oy,
                      int64_t opitch, oracle_level_stats *stats, int max_levels,
                      oracle_region_rec *recs, int64_t rec_cap, int64_t *rec_count)
{
    ask_ctx c;
    memset(&c, 0, sizeof c);
    c.ox = ox;
    c.oy = oy;
    c.opitch = opitch;
    c.reg = reg;
    c.n = n;
    c.maxdwell = maxdwell;
    c.r = r;
    c.B = B;
    c.out = out;
    c.stats = stats;
    c.max_levels = max_levels;
    c.recs = recs;
    c.rec_cap = rec_cap;
    if (maxdwell < 1)
        return 1;
    return run_ask(&c, g, tiles, ntiles, rec_count);
}

int oracle_ask(oracle_region reg, int64_t n, int32_t maxdwell, int g, int r, int B,
               const int32_t *tiles, int64_t ntiles, int32_t *out,
               oracle_level_stats *stats, int max_levels,
               oracle_region_rec *recs, int64_t rec_cap, int64_t *rec_count)
{
    return oracle_ask_window(reg, n, maxdwell, g, r, B, tiles, ntiles, out, 0, 0, n, stats,
                             max_levels, recs, rec_cap, rec_count);
}

int oracle_ask_by_lookup(const int32_t *E, int64_t n, int g, int r, int B,
                         const int32_t *tiles, int64_t ntiles, int32_t *out,
                         oracle_level_stats *stats, int max_levels)
{
    ask_ctx c;
    memset(&c, 0, sizeof c);
    c.n = n;
    c.r = r;
    c.B = B;
    c.lookup = E;
    c.out = out;
    c.opitch = n;
    c.stats = stats;
    c.max_levels = max_levels;
    return run_ask(&c, g, tiles, ntiles, NULL);
}
