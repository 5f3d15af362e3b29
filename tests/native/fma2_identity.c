/* Pin for DESIGN.md R4': the dwell step's imaginary update y = (xy + xy) + ci (two RN float
 * additions, the oracle's literal form) equals fmaf(xy, 2, ci) (one rounding of the
 * exact 2*xy + ci): 2*xy is exact whenever xy + xy does not overflow, and when it does
 * (|xy| >= 2^127) both forms give the same infinity unless |ci| >= 2^103 is large enough to pull
 * the exact sum back below the overflow threshold (or ci is infinite).  So a mismatch needs
 * |xy| >= 2^127, i.e. an orbit that escaped steps earlier: the dwell (the first escape) never
 * changes.  Checked here for random bit patterns (all classes: zeros, subnormals, normals,
 * huge, inf, NaN), pixel-range ci, and the overflow boundary, with glibc's correctly rounded
 * fmaf and the additions compiled without contraction: every mismatch must be of that one
 * kind.  Prints the pairs checked, the (allowed) overflow-cancellation mismatches and the
 * disallowed ones; exits 1 on any disallowed one.
 * Build: gcc -O1 -ffp-contract=off -fno-fast-math fma2_identity.c -lm */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static float f_of(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t u_of(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

static uint64_t s = 0x9e3779b97f4a7c15ull;
static uint32_t rnd(void)
{
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    return (uint32_t)(s >> 16);
}

static volatile float sink_v;
static int same(float a, float b)
{
    if (isnan(a) || isnan(b))
        return isnan(a) && isnan(b);
    return u_of(a) == u_of(b); /* distinguishes +0 / -0 */
}

static long checked = 0, allowed = 0, bad = 0;
static void check(float a, float c)
{
    volatile float t = a + a; /* RN(a + a) */
    volatile float lit = t + c;
    float f = fmaf(a, 2.0f, c);
    ++checked;
    if (!same(lit, f)) {
        /* the one admissible kind: a + a overflows and |c| >= 2^103 (or c infinite) */
        if (fabsf(a) >= 0x1p127f && !isnan(a) && (isinf(c) || fabsf(c) >= 0x1p103f)) {
            ++allowed;
            return;
        }
        if (bad < 10)
            printf("mismatch a=%a c=%a literal=%a fma=%a\n", a, c, (double)lit, (double)f);
        ++bad;
    }
}

/* The dwell (R2/R4) with the literal update and with the fused one. */
static int dwell_lit(float cr, float ci, int md)
{
    volatile float x = 0.f, y = 0.f;
    for (int i = 1; i <= md; ++i) {
        const float x2 = x * x, y2 = y * y, xy = x * y;
        const float t = xy + xy;
        x = (x2 - y2) + cr;
        y = t + ci;
        if (x * x + y * y > 4.0f)
            return i;
    }
    return md;
}
static int dwell_fma(float cr, float ci, int md)
{
    volatile float x = 0.f, y = 0.f;
    for (int i = 1; i <= md; ++i) {
        const float x2 = x * x, y2 = y * y, xy = x * y;
        x = (x2 - y2) + cr;
        y = fmaf(xy, 2.0f, ci);
        if (x * x + y * y > 4.0f)
            return i;
    }
    return md;
}

int main(int argc, char **argv)
{
    /* dwell-level equivalence: pixel-range c (the set's neighbourhood) and arbitrary finite c */
    long dchk = 0, dbad = 0;
    for (int i = 0; i < 200000; ++i) {
        float cr, ci;
        if (i & 1) {
            ci = (float)(-1.3 + 2.6 * (double)(rnd() & 0xffffff) / 16777216.0);
            cr = (float)(-2.1 + 2.7 * (double)(rnd() & 0xffffff) / 16777216.0);
        } else {
            do {
                cr = f_of(rnd());
                ci = f_of(rnd());
            } while (!isfinite(cr) || !isfinite(ci));
        }
        ++dchk;
        if (dwell_lit(cr, ci, 2048) != dwell_fma(cr, ci, 2048)) {
            if (dbad < 10)
                printf("dwell mismatch c=%a%+ai\n", (double)cr, (double)ci);
            ++dbad;
        }
    }
    printf("dwells checked %ld mismatches %ld\n", dchk, dbad);
    if (dbad)
        return 1;

    long n = argc > 1 ? atol(argv[1]) : 20000000L;
    const float edge[] = {0.0f, -0.0f, 1e-45f, -1e-45f, 1.1754942e-38f, 1.17549435e-38f, 1.0f, -1.0f, 2.0f,
                          -2.0f, 1.7014117e38f, 1.7014118e38f, -1.7014118e38f, 3.4028235e38f,
                          -3.4028235e38f, INFINITY, -INFINITY, NAN, 0.5f, 1.9f, -1.9f, 3.9e-39f};
    const int ne = (int)(sizeof edge / sizeof edge[0]);
    for (int i = 0; i < ne; ++i)
        for (int j = 0; j < ne; ++j)
            check(edge[i], edge[j]);
    /* the overflow boundary of a + a: |a| just below / at 2^127 */
    for (int k = -4096; k <= 4096; ++k) {
        const float a = f_of(u_of(1.7014118e38f) + (uint32_t)k);
        for (int j = 0; j < ne; ++j) {
            check(a, edge[j]);
            check(-a, edge[j]);
        }
    }
    for (long i = 0; i < n; ++i) {
        /* random bit patterns for xy; ci from random patterns and the pixel range |ci| < 2 */
        const float a = f_of(rnd());
        const float c = (i & 1) ? f_of(rnd()) : (float)((double)(int32_t)rnd() / 1073741824.0);
        check(a, c);
        /* dwell-like magnitudes: xy in [-8, 8] */
        const float a2 = (float)((double)(int32_t)rnd() / 268435456.0);
        check(a2, c);
    }
    printf("checked %ld overflow_cancellations %ld mismatches %ld\n", checked, allowed, bad);
    return bad != 0;
}
