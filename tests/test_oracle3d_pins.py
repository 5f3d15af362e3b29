"""Pins of the 3-D oracle (oracle/mandel3d_oracle.c; NEXT-4, the paper's k-D extension,
P:549-597; DESIGN.md §12 and readings R15-R17) against things other than itself: the w = 0
slice is the independently pinned 2-D dwell, closed-form orbits (exact fixed points, the
strict escape test, |w|^(2^i) growth), an invariant-disk window and an escape window, the
conjugate symmetry, the k-D OLT size identity |T_i^k| = |G_i| prod r_j, exact volume
tiling, and a second (numpy) implementation of the subdivision recursion on tiny volumes."""
import itertools

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.filterwarnings("ignore")


def test_w0_slice_is_the_2d_dwell():
    # z_0 = w = 0 is the Mandelbrot iteration of the 2-D oracle (pinned in test_oracle_pins)
    for md in (64, 512, 2048):
        for cr in np.linspace(-2.1, 0.6, 37, dtype=np.float32):
            for ci in np.linspace(-1.2, 1.2, 23, dtype=np.float32):
                assert oracle.dwell3(float(cr), float(ci), 0.0, md) == oracle.dwell(float(cr), float(ci), md)


@pytest.mark.parametrize("md", [1, 7, 512, 4096])
def test_closed_form_orbits(md):
    # c = 1/4, w = 1/2: z_1 = 1/4 + 1/4 = 1/2, a fixed point, exact in binary32 -> never escapes
    assert oracle.dwell3(0.25, 0.0, 0.5, md) == md
    # c = -2, w = 2: z_i = 4 - 2 = 2 for every i, |z|^2 = 4 is NOT > 4 (strict test, R2)
    assert oracle.dwell3(-2.0, 0.0, 2.0, md) == md
    # c = -1, w = -1: the 2-cycle -1 -> 0 -> -1 (exact)
    assert oracle.dwell3(-1.0, 0.0, -1.0, md) == md
    # c = 0: z_i = w^(2^i); escape at the first i with w^(2^i) > 2
    assert oracle.dwell3(0.0, 0.0, 1.5, md) == 1                 # 2.25
    assert oracle.dwell3(0.0, 0.0, 1.25, md) == min(2, md)       # 1.5625, 2.44...
    assert oracle.dwell3(0.0, 0.0, 1.0625, md) == min(4, md)     # 1.129, 1.274, 1.624, 2.64
    assert oracle.dwell3(0.0, 0.0, -0.875, md) == md             # |w| < 1: z_i -> 0
    # |c| > 2 escapes at once whatever w in [-1/2, 1/2]: |z_1| >= |c| - w^2 > 2
    assert oracle.dwell3(2.5, 0.5, 0.5, md) == 1
    assert oracle.dwell3(-0.5, 2.6, -0.5, md) == 1


def test_voxel_centres_are_dyadic():
    reg = W.DEFAULT_REGION3
    n = 64
    for (x, y, z) in [(0, 0, 0), (63, 63, 63), (5, 17, 40)]:
        cr, ci, w = oracle.voxel_c(reg, n, x, y, z)
        assert cr == reg[0] + (x + 0.5) * (reg[1] - reg[0]) / n
        assert ci == reg[2] + (y + 0.5) * (reg[3] - reg[2]) / n
        assert w == reg[4] + (z + 0.5) * (reg[5] - reg[4]) / n


def test_closed_form_windows_and_symmetry():
    # |c| <= 1/4 and |w| <= 1/2: the disk |z| <= 1/2 is invariant (1/4 + 1/4), never escapes
    E = oracle.exhaustive3(W.INTERIOR_REGION3, 16, 300)
    assert np.all(E == 300)
    A, st = oracle.ask3(W.INTERIOR_REGION3, 16, 300, 2, 2, 2)
    assert np.all(A == 300) and st[0]["filled"] == 8
    # Re c >= 2.5: |z_1| >= w^2 + Re c > 2
    assert np.all(oracle.exhaustive3(W.ESCAPE_REGION3, 16, 300) == 1)
    # conjugation (w real): the volume over a region symmetric in im is mirror-symmetric in y
    E = oracle.exhaustive3(W.DEFAULT_REGION3, 32, 200)
    assert np.array_equal(E, E[:, ::-1, :])


def _ask3_numpy(E, g, r, B):
    """A second implementation of the 3-D recursion (R17), over a known volume E[z, y, x]."""
    n = E.shape[0]
    out = np.full_like(E, -1)
    stats = {}

    def region(x0, y0, z0, d, lv):
        s = stats.setdefault(lv, dict(regions_in=0, filled=0, subdivided=0, leaves=0))
        s["regions_in"] += 1
        cube = E[z0:z0 + d, y0:y0 + d, x0:x0 + d]
        mask = np.ones((d, d, d), dtype=bool)
        if d > 2:
            mask[1:-1, 1:-1, 1:-1] = False
        surf = cube[mask]
        if np.all(surf == surf[0]):
            out[z0:z0 + d, y0:y0 + d, x0:x0 + d] = surf[0]
            s["filled"] += 1
        elif d // r >= B:
            s["subdivided"] += 1
            h = d // r
            for cz, cy, cx in itertools.product(range(r), repeat=3):
                region(x0 + cx * h, y0 + cy * h, z0 + cz * h, h, lv + 1)
        else:
            out[z0:z0 + d, y0:y0 + d, x0:x0 + d] = cube
            s["leaves"] += 1

    d0 = n // g
    for gz, gy, gx in itertools.product(range(g), repeat=3):
        region(gx * d0, gy * d0, gz * d0, d0, 0)
    return out, [stats[k] for k in sorted(stats)]


@pytest.mark.parametrize("w", list(W.random_small_workloads3(16, seed=W.SEED + 51, max_n=32)),
                         ids=lambda w: w.name)
def test_ask3_against_second_implementation(w):
    E = oracle.exhaustive3(w.region, w.n, w.maxdwell)
    A, st = oracle.ask3(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    B_, st2 = _ask3_numpy(E, w.g, w.r, w.B)
    assert np.array_equal(A, B_)
    assert [{k: s[k] for k in ("regions_in", "filled", "subdivided", "leaves")} for s in st] == st2
    # ASK decisions on computed dwells == the same decisions replayed on the exhaustive volume
    L, stl = oracle.ask3_by_lookup(E, w.g, w.r, w.B)
    assert np.array_equal(A, L) and stl == st


@pytest.mark.parametrize("n,g,r,B", [(64, 2, 2, 4), (64, 4, 2, 2), (64, 1, 4, 4), (32, 2, 4, 2)])
def test_ask3_structure(n, g, r, B):
    md = 200
    A, st = oracle.ask3(W.DEFAULT_REGION3, n, md, g, r, B)
    assert A.min() >= 1 and A.max() <= md
    d = n // g
    covered = 0
    assert st[0]["regions_in"] == g ** 3
    for lv, s in enumerate(st):
        assert s["regions_in"] == s["filled"] + s["subdivided"] + s["leaves"]
        if lv + 1 < len(st):
            # the k-D OLT size: |T_i^k| = |G_i| * prod_j r_j regions at the next level
            assert st[lv + 1]["regions_in"] == s["subdivided"] * r ** 3
        else:
            assert s["subdivided"] == 0
        surf = d ** 3 - max(d - 2, 0) ** 3
        assert s["border_px"] == s["regions_in"] * surf
        assert s["leaf_px"] == s["leaves"] * max(d - 2, 0) ** 3
        covered += (s["filled"] + s["leaves"]) * d ** 3
        d //= r
    assert covered == n ** 3  # terminal regions tile the volume exactly once


def test_ask3_vs_exhaustive_mismatch_is_small():
    n, md = 64, 256
    E = oracle.exhaustive3(W.DEFAULT_REGION3, n, md)
    A, _ = oracle.ask3(W.DEFAULT_REGION3, n, md, 2, 2, 4)
    frac = float((A != E).mean())
    assert frac < 1e-2  # the heuristic may differ where a thin feature slips between surfaces


@pytest.mark.parametrize("n,g,r,B,md", [(32, 2, 2, 4, 200), (64, 4, 2, 2, 100), (32, 2, 4, 2, 64)])
def test_ask3_tile_equals_whole_volume(n, g, r, B, md):
    """oracle.ask3_tile (level-0 cube at a non-zero origin (ox, oy, oz)) equals the matching
    block of the whole-volume recursion and of the independent numpy recursion."""
    region = W.DEFAULT_REGION3
    A, _ = oracle.ask3(region, n, md, g, r, B)
    E = oracle.exhaustive3(region, n, md)
    Np, _ = _ask3_numpy(E, g, r, B)
    d0 = n // g
    for t in range(g ** 3):
        gx, gy, gz = t % g, (t // g) % g, t // (g * g)
        img, _ = oracle.ask3_tile(region, n, md, g, r, B, t)
        sl = (slice(gz * d0, (gz + 1) * d0), slice(gy * d0, (gy + 1) * d0), slice(gx * d0, (gx + 1) * d0))
        assert np.array_equal(img, A[sl]), t
        assert np.array_equal(img, Np[sl]), t
