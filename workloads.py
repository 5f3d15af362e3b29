"""Seeded workload definitions shared by the CUDA path's tests/bench and the oracle.

This module holds ONLY the inputs of the method — complex-plane regions, image sides,
maxdwell and {g, r, B} — and a seeded generator of small random cases.  It contains none
of the method's arithmetic (no pixel mapping, no dwell, no subdivision), so neither side
can borrow the other's implementation through it.

Sources for each configuration (P:NNN = /root/reference/PAPER.md line NNN):
  * default region  -- P:432 prints "[-1.5,-1]x[0.5,1]"; read as the corner pair
                       (-1.5,-1)..(0.5,1), i.e. re in [-1.5,0.5], im in [-1,1] (R1).
  * maxdwell 512    -- P:432 "using a dwell of d=512"; larger maxdwell per BASELINE.json.
  * {g, r, B}       -- P:477-487 sweep space and optima; BASELINE.json configs 1-5.
  * seahorse window -- BASELINE.json config 5 ("zoomed seahorse-valley region"); the exact
                       dyadic window is DESIGN.md reading R9 (SURVEY.md §8(d) C5 proposal).
"""
from __future__ import annotations

import dataclasses
import random
from typing import Iterator, List, Optional, Sequence, Tuple

SEED = 20220605  # the only seed of the run.

# (re_min, re_max, im_min, im_max)
Region = Tuple[float, float, float, float]

DEFAULT_REGION: Region = (-1.5, 0.5, -1.0, 1.0)
SEAHORSE_REGION: Region = (-0.765625, -0.734375, 0.09375, 0.125)
# Closed-form pin windows (SURVEY.md §8(c) "tiny-grid agreement"):
INTERIOR_REGION: Region = (-0.25, 0.125, -0.25, 0.125)  # inside the main cardioid
ESCAPE_REGION: Region = (2.5, 3.5, 2.5, 3.5)  # |c| > 2 everywhere: dwell 1
# Non-dyadic windows (P:432 takes an arbitrary window of the complex plane): their corners
# and pixel pitch are not exact binary fractions, so every pixel centre is rounded.
NONDYADIC_REGIONS: Tuple[Region, ...] = (
    (-0.74531, -0.74419, 0.11273, 0.11385),        # seahorse-valley detail
    (-1.2345678, -0.3456789, 0.0123457, 0.9012345),  # a generic window across the boundary
    (-0.1, 0.3, 0.6, 0.7),                          # non-square: dx != dy
)


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    region: Region
    n: int
    maxdwell: int
    g: int
    r: int
    B: int

    def as_dict(self) -> dict:
        return dataclasses.asdict(self)


# BASELINE.json configs.
C1 = Workload("C1", DEFAULT_REGION, 1024, 512, 4, 2, 32)
C2_N, C2_MAXDWELL = 8192, 2048
C2_G = (2, 4, 8, 16, 32)
C2_R = (2, 4, 8)
C2_B = (16, 32, 64, 128)
C3 = Workload("C3", DEFAULT_REGION, 32768, 2048, 16, 2, 32)
C4 = Workload("C4", DEFAULT_REGION, 65536, 4096, 16, 2, 32)
C5 = Workload("C5", SEAHORSE_REGION, 32768, 2048, 16, 4, 32)

CONFIGS = {w.name: w for w in (C1, C3, C4, C5)}


def c2_sweep() -> List[Workload]:
    """BASELINE.json config 2: g x r x B sweep at n=8192, maxdwell=2048 (60 points)."""
    out = []
    for g in C2_G:
        for r in C2_R:
            for B in C2_B:
                if g * B <= C2_N:
                    out.append(Workload(f"C2_g{g}_r{r}_B{B}", DEFAULT_REGION, C2_N,
                                        C2_MAXDWELL, g, r, B))
    return out


def _pow2s(lo: int, hi: int) -> List[int]:
    v, out = lo, []
    while v <= hi:
        out.append(v)
        v *= 2
    return out


def random_small_workloads(count: int, seed: int = SEED, max_n: int = 512,
                           regions: Optional[Sequence[Region]] = None) -> Iterator[Workload]:
    """Seeded random small cases: powers of two with g*B <= n, r >= 2, B >= 2.

    Regions are drawn from dyadic sub-windows of the default region (pixel centres exact in
    FP32), the named windows, and NON-dyadic windows (NONDYADIC_REGIONS), where the pixel
    mapping of DESIGN.md R3 rounds and its operation order decides the bits.
    """
    rng = random.Random(seed)
    if regions is None:
        regions = [DEFAULT_REGION, SEAHORSE_REGION,
                   (-1.0, 0.0, 0.0, 1.0), (-0.875, -0.625, 0.0, 0.25),
                   (-1.5, -1.25, -0.125, 0.125), (0.25, 0.5, -0.125, 0.125)] + list(NONDYADIC_REGIONS)
    k = 0
    while k < count:
        n = rng.choice(_pow2s(8, max_n))
        g = rng.choice(_pow2s(1, n // 2))
        B = rng.choice(_pow2s(2, max(2, n // g)))
        if g * B > n:
            continue
        r = rng.choice([2, 4, 8])
        maxdwell = rng.choice([1, 2, 7, 64, 100, 256, 512, 1000])
        yield Workload(f"rand{k}", rng.choice(list(regions)), n, maxdwell, g, r, B)
        k += 1


# ------------------------------------------------------------------ k = 3 (NEXT-4)
# The paper sketches ASK on k-orthotopes without a 3-D workload; R15-R17 fix one:
# the (c_re, c_im, w) slice of the quadratic family's parameter space, z_0 = w (w = 0 is the
# Mandelbrot set).  Regions are (re_min, re_max, im_min, im_max, w_min, w_max), dyadic so the
# voxel centres are exact in FP32.
Region3 = Tuple[float, float, float, float, float, float]

DEFAULT_REGION3: Region3 = (-1.5, 0.5, -1.0, 1.0, -0.5, 0.5)
INTERIOR_REGION3: Region3 = (-0.125, 0.125, -0.125, 0.125, -0.25, 0.25)  # |c| <= 1/4, |w| <= 1/2
ESCAPE_REGION3: Region3 = (2.5, 3.5, 2.5, 3.5, -0.5, 0.5)                # dwell 1 everywhere


@dataclasses.dataclass(frozen=True)
class Workload3:
    name: str
    region: Region3
    n: int
    maxdwell: int
    g: int
    r: int
    B: int

    def as_dict(self) -> dict:
        return dataclasses.asdict(self)


# Measured 3-D configurations (tools/bench3d.py): a 512^3 (512 MiB) and a 1024^3 (4 GiB)
# volume; leaves of side 8 (4 levels) and 16.
V1 = Workload3("V1", DEFAULT_REGION3, 512, 512, 8, 2, 8)
V2 = Workload3("V2", DEFAULT_REGION3, 1024, 1024, 8, 2, 16)
CONFIGS3 = {w.name: w for w in (V1, V2)}


def random_small_workloads3(count: int, seed: int = SEED, max_n: int = 64) -> Iterator[Workload3]:
    """Seeded random small 3-D cases (powers of two, g*B <= n, r in {2, 4})."""
    rng = random.Random(seed)
    regions = [DEFAULT_REGION3, (-1.0, 0.0, 0.0, 1.0, -0.25, 0.25), (-0.875, -0.625, 0.0, 0.25, 0.0, 0.25),
               (-1.5, -1.25, -0.125, 0.125, -0.5, 0.0), (0.25, 0.5, -0.125, 0.125, -0.0625, 0.0625)]
    k = 0
    while k < count:
        n = rng.choice(_pow2s(4, max_n))
        g = rng.choice(_pow2s(1, n // 2))
        B = rng.choice(_pow2s(2, max(2, n // g)))
        if g * B > n:
            continue
        r = rng.choice([2, 4])
        maxdwell = rng.choice([1, 2, 7, 64, 100, 256])
        yield Workload3(f"v{k}", rng.choice(regions), n, maxdwell, g, r, B)
        k += 1
