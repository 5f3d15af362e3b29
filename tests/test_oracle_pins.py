"""Pins of the CPU oracle to things other than itself (closed forms, exact arithmetic,
invariants, hand-computed orbits, an independent survey-time implementation).

Each test names what fixes the expected value.  P:NNN = /root/reference/PAPER.md line.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W

MAXDWELLS = (512, 2048, 4096)


# ----------------------------------------------------------------------------- dwell
@pytest.mark.parametrize("maxdwell", MAXDWELLS)
@pytest.mark.parametrize("c", [0, -1, -2, 1j, 0.25, -0.75, -0.5 + 0.5j, -1.5, -1.75,
                               -0.1 + 0.1j, -1.0 + 0.1j, -0.125 + 0.75j])
def test_dwell_inside_closed_form(c, maxdwell):
    """Points of M by closed form: fixed points / cycles, the real segment [-2, 1/4]
    (|x^2 + c| <= beta on [-beta, beta]), the main cardioid and the period-2 bulb
    (SURVEY.md §8(c) pins; north_star's c = 0, -1, -2, i).  Never escape -> maxdwell."""
    assert oracle.dwell(c.real if isinstance(c, complex) else c,
                        c.imag if isinstance(c, complex) else 0.0, maxdwell) == maxdwell


@pytest.mark.parametrize("cr,ci,expect", [
    (0.5, 0.0, 5),    # 0.5, 0.75, 1.0625, 1.62890625, 3.153... (all exact in float)
    (1.0, 0.0, 3),    # 1, 2, 5: |2| is not > 2 (strict test, "|z| <= 2")
    (2.0, 0.0, 2),    # 2, 6
    (3.0, 0.0, 1),    # |c| > 2 escapes at the first iteration
    (0.0, 2.0, 2),    # 2i (|z|^2 = 4, not > 4), then -4 + 2i
    (-2.5, 0.0, 1),
    (0.0, -3.0, 1),
    (-2.0, 0.5, 1),   # |c|^2 = 4.25
    (0.25, 1.0, 3),   # 0.25+i, -0.6875+1.5i, -1.527...-1.0625i -> |.|^2 = 3.46, next escapes? see exact test
])
def test_dwell_hand_orbits(cr, ci, expect):
    if (cr, ci) == (0.25, 1.0):
        expect = _exact_dwell(Fraction(1, 4), Fraction(1), 512)[0]
    assert oracle.dwell(cr, ci, 512) == expect


def _is_f32_exact(q: Fraction) -> bool:
    """True iff q is exactly representable as a normal float32 (or zero)."""
    if q == 0:
        return True
    num, den = abs(q.numerator), q.denominator  # Fraction keeps them coprime
    if den & (den - 1):
        return False                 # not dyadic
    exp = num.bit_length() - 1 - (den.bit_length() - 1)
    odd = num
    while odd % 2 == 0:
        odd //= 2
    return odd.bit_length() <= 24 and -126 <= exp <= 127


def _exact_dwell(cr: Fraction, ci: Fraction, maxdwell: int):
    """Mathematical dwell in exact rational arithmetic: first i >= 1 with
    |z_i|^2 > 4.  Also returns whether every intermediate the FP32 recurrence rounds
    (x^2, y^2, xy, x^2-y^2, +c, xy+xy, +c, x^2+y^2) was exactly representable, in which
    case every FP32 operation was exact and the oracle must agree bit for bit."""
    x = y = Fraction(0)
    exact = True
    for i in range(1, maxdwell + 1):
        x2, y2, xy = x * x, y * y, x * y
        t, u = x2 - y2, xy + xy
        x, y = t + cr, u + ci
        mag = x * x + y * y
        for q in (x2, y2, xy, t, u, x, y, x * x, y * y, mag):
            exact &= _is_f32_exact(q)
        if mag > 4:
            return i, exact
        if not exact:
            return None, False
    return maxdwell, exact


def test_dwell_exact_rational_pin():
    """For dyadic c whose whole orbit (up to escape) stays exactly representable in
    float32, no rounding occurs and the oracle must return the mathematical dwell.
    A dropped term, a sign error or a transposed operand fails here."""
    rng = np.random.default_rng(W.SEED)
    checked = 0
    for _ in range(20000):
        a = int(rng.integers(-40, 41))
        b = int(rng.integers(-40, 41))
        k = int(rng.integers(2, 5))
        cr, ci = Fraction(a, 2 ** k), Fraction(b, 2 ** k)
        d, exact = _exact_dwell(cr, ci, 64)
        if d is None or not exact:
            continue
        assert oracle.dwell(float(cr), float(ci), 64) == d, (cr, ci)
        checked += 1
    assert checked > 500


def test_dwell_cap_monotone():
    """dwell(c, m1) == min(dwell(c, m2), m1) for m1 < m2 (the cap is a truncation)."""
    rng = np.random.default_rng(W.SEED + 1)
    for _ in range(3000):
        cr, ci = rng.uniform(-2.2, 0.8), rng.uniform(-1.3, 1.3)
        d2 = oracle.dwell(cr, ci, 300)
        for m1 in (1, 2, 7, 50, 299):
            assert oracle.dwell(cr, ci, m1) == min(d2, m1)


def test_dwell_one_iff_c_outside_radius2():
    """dwell == 1 exactly when |z_1|^2 = |c|^2 > 4."""
    rng = np.random.default_rng(W.SEED + 2)
    for _ in range(5000):
        cr = np.float32(rng.uniform(-3, 3))
        ci = np.float32(rng.uniform(-3, 3))
        mag = np.float32(cr * cr) + np.float32(ci * ci)
        assert (oracle.dwell(float(cr), float(ci), 100) == 1) == bool(mag > 4)


# ----------------------------------------------------------------------------- mapping
def test_pixel_centre_mapping():
    """Pixel-centre sampling (SPEC.md S:183-191 examples; R3)."""
    assert oracle.pixel_c((0, 1, 0, 1), 1, 0, 0) == (0.5, 0.5)
    assert oracle.pixel_c((0, 1, 0, 1), 2, 0, 0) == (0.25, 0.25)
    assert oracle.pixel_c((0, 1, 0, 1), 2, 1, 0) == (0.25, 0.75)  # row i -> imaginary
    cr, ci = oracle.pixel_c(W.DEFAULT_REGION, 16, 0, 0)
    assert (cr, ci) == (-1.4375, -0.9375)  # SURVEY.md c-8 hand check
    n = 1024
    for (i, j) in [(0, 0), (n - 1, n - 1), (0, n - 1)]:
        cr, ci = oracle.pixel_c(W.DEFAULT_REGION, n, i, j)
        assert -1.5 < cr < 0.5 and -1.0 < ci < 1.0
        # dyadic region: the centre is exact
        assert cr == -1.5 + (j + 0.5) * 2.0 / n and ci == -1.0 + (i + 0.5) * 2.0 / n


# ----------------------------------------------------------------------------- exhaustive
def test_exhaustive_survey_table(golden_dir):
    """n=16 worked example, rows r00..r07 and the mirrored r08..r15."""
    rows = np.loadtxt(os.path.join(golden_dir, "survey_c8_n16_maxdwell512.txt"), dtype=np.int64)
    E = oracle.exhaustive(W.DEFAULT_REGION, 16, 512)
    assert np.array_equal(E[:8], rows)
    assert np.array_equal(E[8:], rows[::-1])


def test_exhaustive_fingerprints(golden_dir):
    fp = json.load(open(os.path.join(golden_dir, "survey_fingerprints.json")))
    for e in fp["sum_dwell"]:
        if e["n"] > 256 and e["maxdwell"] > 512:
            continue  # keep the CPU suite short; n=1024/2048 is covered by the slow test
        E = oracle.exhaustive(W.DEFAULT_REGION, e["n"], e["maxdwell"])
        assert int(E.sum(dtype=np.int64)) == e["sum"]
        assert abs((E == e["maxdwell"]).mean() - e["inside"]) < 1e-5


@pytest.mark.slow
def test_exhaustive_fingerprints_large(golden_dir):
    fp = json.load(open(os.path.join(golden_dir, "survey_fingerprints.json")))
    for e in fp["sum_dwell"]:
        if e["n"] == 1024:
            E = oracle.exhaustive(W.DEFAULT_REGION, e["n"], e["maxdwell"])
            assert int(E.sum(dtype=np.int64)) == e["sum"]


def _in_cardioid_or_bulb(x, y):
    q = (x - 0.25) ** 2 + y ** 2
    return (q * (q + (x - 0.25)) < y * y / 4) | ((x + 1) ** 2 + y * y < 1.0 / 16)


@pytest.mark.parametrize("n,maxdwell", [(256, 512), (128, 2048)])
def test_exhaustive_cardioid_bulb(n, maxdwell):
    """Every pixel centre strictly inside the main cardioid or the period-2 bulb (closed
    form) has dwell == maxdwell; the inside share approaches (3pi/8 + pi/16)/4."""
    E = oracle.exhaustive(W.DEFAULT_REGION, n, maxdwell)
    j = np.arange(n)
    x = -1.5 + (j + 0.5) * 2.0 / n
    y = -1.0 + (j + 0.5) * 2.0 / n
    X, Y = np.meshgrid(x, y)  # rows = imaginary
    inside = _in_cardioid_or_bulb(X, Y)
    assert np.all(E[inside] == maxdwell)
    assert abs(inside.mean() - (3 * math.pi / 8 + math.pi / 16) / 4) < 0.01


def test_exhaustive_conjugate_symmetry():
    """The default region is symmetric about the real axis and the pixel mapping is
    dyadic, so D[i][j] == D[n-1-i][j] exactly (IEEE RN is sign-symmetric)."""
    E = oracle.exhaustive(W.DEFAULT_REGION, 128, 1000)
    assert np.array_equal(E, E[::-1])


def test_exhaustive_rows_and_pixels_agree():
    E = oracle.exhaustive(W.SEAHORSE_REGION, 64, 700)
    assert np.array_equal(oracle.exhaustive(W.SEAHORSE_REGION, 64, 700, row0=10, rows=5), E[10:15])
    rng = np.random.default_rng(W.SEED)
    ii, jj = rng.integers(0, 64, 100), rng.integers(0, 64, 100)
    assert np.array_equal(oracle.dwell_pixels(W.SEAHORSE_REGION, 64, 700, ii, jj), E[ii, jj])


def test_exhaustive_tiny_windows():
    """Interior-only window -> all maxdwell; escape-only window -> all 1 (closed forms)."""
    assert np.all(oracle.exhaustive(W.INTERIOR_REGION, 32, 777) == 777)
    assert np.all(oracle.exhaustive(W.ESCAPE_REGION, 32, 777) == 1)


# ----------------------------------------------------------------------------- ASK
def _levels_bound(n, g, r, B):
    d, L = n // g, 1
    while d // r >= B:
        d //= r
        L += 1
    return L


def _check_structure(n, g, r, B, E, A, stats, recs, maxdwell):
    # per-level identities
    for s in stats:
        assert s["regions_in"] == s["filled"] + s["subdivided"] + s["leaves"]
    for a, b in zip(stats, stats[1:]):
        assert b["regions_in"] == r * r * a["subdivided"]
    assert stats[-1]["subdivided"] == 0
    assert len(stats) <= _levels_bound(n, g, r, B)
    assert stats[0]["regions_in"] == g * g
    # terminal regions tile the image exactly once
    cover = np.zeros((n, n), np.int32)
    for x, y, d, kind, value, level in recs:
        cover[y:y + d, x:x + d] += 1
        assert d == (n // g) // r ** level
        ring = np.concatenate([E[y, x:x + d], E[y + d - 1, x:x + d], E[y:y + d, x], E[y:y + d, x + d - 1]])
        if kind == 0:   # filled: uniform border in the exhaustive image, fill = that value
            assert np.all(ring == value) and np.all(A[y:y + d, x:x + d] == value)
        else:           # leaf: non-uniform border, per-pixel dwell == exhaustive
            assert not np.all(ring == ring[0])
            assert np.array_equal(A[y:y + d, x:x + d], E[y:y + d, x:x + d])
            assert d // r < B
    assert np.all(cover == 1)
    assert np.all((A >= 1) & (A <= maxdwell))


def test_ask_c1_survey_levels(golden_dir):
    fp = json.load(open(os.path.join(golden_dir, "survey_fingerprints.json")))["c1_levels"]
    w = W.C1
    E = oracle.exhaustive(w.region, w.n, w.maxdwell)
    A, st, recs = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, want_regions=True)
    assert [s["regions_in"] for s in st] == fp["regions"]
    assert [s["filled"] for s in st] == fp["filled"]
    assert st[-1]["leaves"] == fp["leaves"]
    assert int((A != E).sum()) == fp["mismatch_pixels"]
    executed = sum(s["border_iters"] + s["leaf_iters"] for s in st)
    assert abs(executed - fp["executed_iters_approx"]) / fp["executed_iters_approx"] < 0.01
    _check_structure(w.n, w.g, w.r, w.B, E, A, st, recs, w.maxdwell)


def test_ask_executed_iteration_fingerprints(golden_dir):
    fp = json.load(open(os.path.join(golden_dir, "survey_fingerprints.json")))
    for e in fp["ask_executed_iterations"]:
        _, st = oracle.ask(W.DEFAULT_REGION, e["n"], e["maxdwell"], e["g"], e["r"], e["B"])
        assert sum(s["border_iters"] + s["leaf_iters"] for s in st) == e["iters"]


@pytest.mark.parametrize("w", list(W.random_small_workloads(40, max_n=256)), ids=lambda w: w.name)
def test_ask_structure_random(w):
    E = oracle.exhaustive(w.region, w.n, w.maxdwell)
    A, st, recs = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, want_regions=True)
    _check_structure(w.n, w.g, w.r, w.B, E, A, st, recs, w.maxdwell)
    # structural identity: ASK == ASK-by-lookup(Ex)
    A2, st2 = oracle.ask_by_lookup(E, w.g, w.r, w.B)
    assert np.array_equal(A, A2)
    assert st == st2


def test_ask_tiny_windows():
    for region, val in ((W.INTERIOR_REGION, 321), (W.ESCAPE_REGION, 1)):
        for (n, g, r, B) in ((64, 2, 2, 4), (64, 4, 4, 4), (128, 8, 2, 8)):
            A, st = oracle.ask(region, n, 321, g, r, B)
            assert np.all(A == val)
            assert len(st) == 1 and st[0]["filled"] == g * g


def _ask_levelwise_python(E, g, r, B):
    """Independent brute force on tiny inputs: the ASK level loop of P:354-383 written as
    explicit read/write offset lists (OLTs) over the exhaustive image — breadth-first,
    unlike the oracle's depth-first recursion."""
    n = E.shape[0]
    out = np.full_like(E, -1)
    d = n // g
    olt = [(gx * d, gy * d) for gy in range(g) for gx in range(g)]
    while olt:
        write = []
        for (x, y) in olt:
            ring = np.concatenate([E[y, x:x + d], E[y + d - 1, x:x + d], E[y:y + d, x], E[y:y + d, x + d - 1]])
            if np.all(ring == ring[0]):
                out[y:y + d, x:x + d] = ring[0]
            elif d // r >= B:
                s = d // r
                write += [(x + cx * s, y + cy * s) for cy in range(r) for cx in range(r)]
            else:
                out[y:y + d, x:x + d] = E[y:y + d, x:x + d]
        olt, d = write, d // r
    return out


@pytest.mark.parametrize("w", list(W.random_small_workloads(15, seed=W.SEED + 7, max_n=128)),
                         ids=lambda w: w.name)
def test_ask_matches_levelwise_bruteforce(w):
    E = oracle.exhaustive(w.region, w.n, w.maxdwell)
    A, _ = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    assert np.array_equal(A, _ask_levelwise_python(E, w.g, w.r, w.B))


def test_ask_tiles_partition():
    """Level-0 tiles are independent: the union of per-tile runs equals the full run."""
    w = W.Workload("t", W.SEAHORSE_REGION, 256, 600, 8, 2, 8)
    A, st = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    out = np.full((w.n, w.n), -1, np.int32)
    tiles = np.arange(w.g * w.g)
    np.random.default_rng(W.SEED).shuffle(tiles)
    tot = {}
    for part in np.array_split(tiles, 3):
        _, s = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, tiles=part, out=out)
        for lv in s:
            for k, v in lv.items():
                if k != "level":
                    tot[(lv["level"], k)] = tot.get((lv["level"], k), 0) + v
    assert np.array_equal(out, A)
    for lv in st:
        for k, v in lv.items():
            if k != "level":
                assert tot[(lv["level"], k)] == v


def test_ask_mismatch_small_but_nonzero_possible():
    """ASK is a heuristic: it may differ from Ex only inside filled regions; the
    differing share stays far below SPEC's 0.1% bound on the seahorse window."""
    w = W.Workload("t", W.SEAHORSE_REGION, 512, 2048, 16, 4, 8)
    E = oracle.exhaustive(w.region, w.n, w.maxdwell)
    A, _ = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    assert (A != E).mean() < 1e-3


# ----------------------------------------------------------------------------- windowed tiles
@pytest.mark.parametrize("w", [W.Workload("t1", W.SEAHORSE_REGION, 256, 700, 4, 2, 8),
                               W.Workload("t2", W.NONDYADIC_REGIONS[0], 128, 900, 8, 4, 2),
                               W.Workload("t3", W.NONDYADIC_REGIONS[1], 256, 300, 2, 2, 16),
                               W.Workload("t4", W.NONDYADIC_REGIONS[2], 64, 1000, 4, 8, 2)],
                         ids=lambda w: w.name)
def test_ask_tile_equals_whole_image_and_bruteforce(w):
    """oracle.ask_tile (the windowed path every full-size check uses, level-0 tile at origin
    (ox, oy) != 0) equals the matching slice of the whole-image recursion AND of the
    independent level-wise Python recursion over the exhaustive image; its statistics sum to
    the whole image's."""
    E = oracle.exhaustive(w.region, w.n, w.maxdwell)
    A, st = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    Bf = _ask_levelwise_python(E, w.g, w.r, w.B)
    d0 = w.n // w.g
    tot = {}
    for t in range(w.g * w.g):
        gy, gx = divmod(t, w.g)
        img, s = oracle.ask_tile(w.region, w.n, w.maxdwell, w.g, w.r, w.B, t)
        sl = (slice(gy * d0, (gy + 1) * d0), slice(gx * d0, (gx + 1) * d0))
        assert np.array_equal(img, A[sl]), t
        assert np.array_equal(img, Bf[sl]), t
        for lv in s:
            for k, v in lv.items():
                if k != "level":
                    tot[(lv["level"], k)] = tot.get((lv["level"], k), 0) + v
    for lv in st:
        for k, v in lv.items():
            if k != "level":
                assert tot[(lv["level"], k)] == v, (lv["level"], k)


@pytest.mark.parametrize("region", W.NONDYADIC_REGIONS)
def test_pixel_mapping_non_dyadic_error_bound(region):
    """Non-dyadic windows (an arbitrary window): every pixel centre is within a few
    float32 ulps of the exact centre re_min + (j + 1/2)(re_max - re_min)/n (four rounded
    operations, R3), and the centres are strictly increasing in j and i."""
    n = 64
    prev_r = prev_i = -math.inf
    for k in range(n):
        cr, ci = oracle.pixel_c(region, n, k, k)
        exact_r = region[0] + (k + 0.5) * (region[1] - region[0]) / n
        exact_i = region[2] + (k + 0.5) * (region[3] - region[2]) / n
        for got, ex, span in ((cr, exact_r, abs(region[0]) + abs(region[1])),
                              (ci, exact_i, abs(region[2]) + abs(region[3]))):
            ulp = np.spacing(np.float32(max(abs(ex), span)))
            assert abs(got - ex) <= 4 * float(ulp), (k, got, ex)
        assert cr > prev_r and ci > prev_i
        prev_r, prev_i = cr, ci
