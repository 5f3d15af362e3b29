"""CPU oracle for the ASK Mandelbrot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this package.  The product package (paper_2206_02255_b200) never imports it
and shares no code with it; the only shared module is the input definitions in
workloads.py, which hold none of the method's arithmetic.

Contents:
  * mandel_oracle.c  -- plain single-threaded C: dwell, Ex,
                        recursive Mariani-Silver / ASK, ASK-by-lookup.
  * montecarlo.py    -- Bernoulli subdivision-tree simulation of the cost model's work
                        (P:120-182), the oracle for costmodel.W_S / W_SSD.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
import threading
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mandel_oracle.c")
_SRC3 = os.path.join(_HERE, "mandel3d_oracle.c")  # k = 3 extension
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]

MAX_LEVELS = 32

_lock = threading.Lock()
_lib: Optional[ctypes.CDLL] = None


def source_sha() -> str:
    """SHA-256 of the oracle's C sources and flags: the version key of every cached oracle
    result (oracle/cache.py) and of the rebuild check below."""
    h = hashlib.sha256()
    for p in (_SRC, _SRC3):
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(CFLAGS).encode())
    return h.hexdigest()


def build(force: bool = False) -> str:
    """Compile liboracle.so with contraction off (R4); rebuilt whenever the source
    hash recorded beside it differs."""
    digest = source_sha()
    stamp = _LIB + ".srchash"
    fresh = os.path.exists(_LIB) and os.path.exists(stamp) and open(stamp).read().strip() == digest
    if force or not fresh:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, _SRC3])
        os.replace(tmp, _LIB)
        with open(stamp, "w") as f:
            f.write(digest + "\n")
    return _LIB


class Region(ctypes.Structure):
    _fields_ = [("re_min", ctypes.c_double), ("re_max", ctypes.c_double),
                ("im_min", ctypes.c_double), ("im_max", ctypes.c_double)]


class LevelStats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in (
        "regions_in", "filled", "subdivided", "leaves",
        "border_px", "border_iters", "leaf_px", "leaf_iters")]


class Region3(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("re_min", "re_max", "im_min", "im_max", "w_min", "w_max")]


class RegionRec(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in ("x", "y", "d", "kind", "value", "level")]


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            P = ctypes.POINTER
            i32p, i64p = P(ctypes.c_int32), P(ctypes.c_int64)
            L.oracle_dwell.restype = ctypes.c_int32
            L.oracle_dwell.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_int32]
            L.oracle_pixel_c.restype = None
            L.oracle_pixel_c.argtypes = [Region, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         P(ctypes.c_float), P(ctypes.c_float)]
            L.oracle_exhaustive_rows.restype = None
            L.oracle_exhaustive_rows.argtypes = [Region, ctypes.c_int64, ctypes.c_int32,
                                                 ctypes.c_int64, ctypes.c_int64, i32p]
            L.oracle_dwell_pixels.restype = None
            L.oracle_dwell_pixels.argtypes = [Region, ctypes.c_int64, ctypes.c_int32, i64p, i64p,
                                              ctypes.c_int64, i32p]
            L.oracle_ask.restype = ctypes.c_int
            L.oracle_ask.argtypes = [Region, ctypes.c_int64, ctypes.c_int32, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, i32p, ctypes.c_int64, i32p,
                                     P(LevelStats), ctypes.c_int, P(RegionRec), ctypes.c_int64,
                                     i64p]
            L.oracle_ask_window.restype = ctypes.c_int
            L.oracle_ask_window.argtypes = [Region, ctypes.c_int64, ctypes.c_int32, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, i32p, ctypes.c_int64, i32p,
                                            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                            P(LevelStats), ctypes.c_int, P(RegionRec),
                                            ctypes.c_int64, i64p]
            L.oracle_ask_by_lookup.restype = ctypes.c_int
            L.oracle_ask_by_lookup.argtypes = [i32p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, i32p, ctypes.c_int64, i32p,
                                               P(LevelStats), ctypes.c_int]
            # k = 3 (mandel3d_oracle.c)
            L.oracle3_dwell.restype = ctypes.c_int32
            L.oracle3_dwell.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_int32]
            L.oracle3_voxel_c.restype = None
            L.oracle3_voxel_c.argtypes = [Region3, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                          P(ctypes.c_float), P(ctypes.c_float), P(ctypes.c_float)]
            L.oracle3_exhaustive_slices.restype = None
            L.oracle3_exhaustive_slices.argtypes = [Region3, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64,
                                                    ctypes.c_int64, i32p]
            L.oracle3_ask_window.restype = ctypes.c_int
            L.oracle3_ask_window.argtypes = [Region3, ctypes.c_int64, ctypes.c_int32, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, i32p, ctypes.c_int64, i32p, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                             P(LevelStats), ctypes.c_int]
            L.oracle3_ask_by_lookup.restype = ctypes.c_int
            L.oracle3_ask_by_lookup.argtypes = [i32p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                i32p, P(LevelStats), ctypes.c_int]
            _lib = L
    return _lib


def _i32(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _i64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def dwell(cr: float, ci: float, maxdwell: int) -> int:
    """Dwell of c = cr + i ci (both rounded to float32 first)."""
    return int(lib().oracle_dwell(cr, ci, maxdwell))


def pixel_c(region, n: int, i: int, j: int) -> Tuple[float, float]:
    cr, ci = ctypes.c_float(), ctypes.c_float()
    lib().oracle_pixel_c(Region(*region), n, i, j, ctypes.byref(cr), ctypes.byref(ci))
    return cr.value, ci.value


def exhaustive(region, n: int, maxdwell: int, row0: int = 0, rows: Optional[int] = None) -> np.ndarray:
    """Ex image rows [row0, row0+rows) as int32 (rows x n)."""
    rows = n - row0 if rows is None else rows
    out = np.empty((rows, n), dtype=np.int32)
    lib().oracle_exhaustive_rows(Region(*region), n, maxdwell, row0, rows, _i32(out))
    return out


def dwell_pixels(region, n: int, maxdwell: int, ii, jj) -> np.ndarray:
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    out = np.empty(ii.shape, dtype=np.int32)
    lib().oracle_dwell_pixels(Region(*region), n, maxdwell, _i64(ii), _i64(jj), ii.size, _i32(out))
    return out


def _stats_list(st, levels: int) -> list:
    out = []
    for lv in range(levels):
        s = st[lv]
        d = {k: int(getattr(s, k)) for k, _ in LevelStats._fields_}
        if d["regions_in"] == 0:
            break
        d["level"] = lv
        out.append(d)
    return out


def ask(region, n: int, maxdwell: int, g: int, r: int, B: int,
        tiles: Optional[Sequence[int]] = None, out: Optional[np.ndarray] = None,
        want_regions: bool = False):
    """Recursive ASK (Mariani-Silver) image.  Returns (image, level_stats[, region_recs]).

    With `tiles`, only those level-0 tiles (canonical k = gy*g + gx) are computed; pixels
    outside them keep the value they have in `out` (default: -1)."""
    L = lib()
    if out is None:
        out = np.full((n, n), -1, dtype=np.int32)
    st = (LevelStats * MAX_LEVELS)()
    t_arr = None if tiles is None else np.ascontiguousarray(tiles, dtype=np.int32)
    recs = None
    cap = 0
    cnt = ctypes.c_int64(0)
    if want_regions:
        cap = 4 * n * n // max(1, B * B) + 16
        recs = (RegionRec * cap)()
    rc = L.oracle_ask(Region(*region), n, maxdwell, g, r, B,
                      None if t_arr is None else _i32(t_arr), 0 if t_arr is None else t_arr.size,
                      _i32(out), st, MAX_LEVELS, recs, cap, ctypes.byref(cnt))
    if rc != 0:
        raise ValueError(f"oracle_ask failed rc={rc}")
    stats = _stats_list(st, MAX_LEVELS)
    if want_regions:
        arr = np.ctypeslib.as_array(recs)[: cnt.value]
        recs_np = np.array([tuple(x) for x in arr], dtype=np.int64).reshape(-1, 6)
        return out, stats, recs_np
    return out, stats


def ask_tile(region, n: int, maxdwell: int, g: int, r: int, B: int, tile: int):
    """ASK of a single level-0 tile into a (d0, d0) array (memory-light for large n).
    Returns (tile image, level_stats)."""
    d0 = n // g
    gy, gx = divmod(int(tile), g)
    out = np.full((d0, d0), -1, dtype=np.int32)
    st = (LevelStats * MAX_LEVELS)()
    t_arr = np.array([tile], dtype=np.int32)
    cnt = ctypes.c_int64(0)
    rc = lib().oracle_ask_window(Region(*region), n, maxdwell, g, r, B, _i32(t_arr), 1, _i32(out),
                                 gx * d0, gy * d0, d0, st, MAX_LEVELS, None, 0, ctypes.byref(cnt))
    if rc != 0:
        raise ValueError(f"oracle_ask_window failed rc={rc}")
    return out, _stats_list(st, MAX_LEVELS)


def ask_by_lookup(E: np.ndarray, g: int, r: int, B: int, tiles: Optional[Sequence[int]] = None):
    """ASK decisions replayed over an exhaustive image E."""
    E = np.ascontiguousarray(E, dtype=np.int32)
    n = E.shape[0]
    out = np.full((n, n), -1, dtype=np.int32)
    st = (LevelStats * MAX_LEVELS)()
    t_arr = None if tiles is None else np.ascontiguousarray(tiles, dtype=np.int32)
    rc = lib().oracle_ask_by_lookup(_i32(E), n, g, r, B,
                                    None if t_arr is None else _i32(t_arr),
                                    0 if t_arr is None else t_arr.size, _i32(out), st, MAX_LEVELS)
    if rc != 0:
        raise ValueError(f"oracle_ask_by_lookup failed rc={rc}")
    return out, _stats_list(st, MAX_LEVELS)


# ------------------------------------------------------------------------ k = 3
def dwell3(cr: float, ci: float, w: float, maxdwell: int) -> int:
    """Dwell of c = cr + i ci from z_0 = w (R15; all three rounded to float32)."""
    return int(lib().oracle3_dwell(cr, ci, w, maxdwell))


def voxel_c(region3, n: int, x: int, y: int, z: int) -> Tuple[float, float, float]:
    cr, ci, w = ctypes.c_float(), ctypes.c_float(), ctypes.c_float()
    lib().oracle3_voxel_c(Region3(*region3), n, x, y, z, ctypes.byref(cr), ctypes.byref(ci), ctypes.byref(w))
    return cr.value, ci.value, w.value


def exhaustive3(region3, n: int, maxdwell: int, z0: int = 0, nz: Optional[int] = None) -> np.ndarray:
    """Exhaustive 3-D dwell volume, z-slices [z0, z0+nz), as int32 (nz, n, n) indexed [z, y, x]."""
    nz = n - z0 if nz is None else nz
    out = np.empty((nz, n, n), dtype=np.int32)
    lib().oracle3_exhaustive_slices(Region3(*region3), n, maxdwell, z0, nz, _i32(out))
    return out


def ask3(region3, n: int, maxdwell: int, g: int, r: int, B: int):
    """Recursive 3-D ASK volume [z, y, x] and its per-level statistics."""
    out = np.full((n, n, n), -1, dtype=np.int32)
    st = (LevelStats * MAX_LEVELS)()
    rc = lib().oracle3_ask_window(Region3(*region3), n, maxdwell, g, r, B, None, 0, _i32(out), 0, 0, 0, n, n,
                                  st, MAX_LEVELS)
    if rc != 0:
        raise ValueError(f"oracle3_ask_window failed rc={rc}")
    return out, _stats_list(st, MAX_LEVELS)


def ask3_tile(region3, n: int, maxdwell: int, g: int, r: int, B: int, tile: int):
    """3-D ASK of one level-0 cube (k = (gz*g + gy)*g + gx) into a (d0, d0, d0) array."""
    d0 = n // g
    gx, gy, gz = tile % g, (tile // g) % g, tile // (g * g)
    out = np.full((d0, d0, d0), -1, dtype=np.int32)
    st = (LevelStats * MAX_LEVELS)()
    t_arr = np.array([tile], dtype=np.int32)
    rc = lib().oracle3_ask_window(Region3(*region3), n, maxdwell, g, r, B, _i32(t_arr), 1, _i32(out),
                                  gx * d0, gy * d0, gz * d0, d0, d0, st, MAX_LEVELS)
    if rc != 0:
        raise ValueError(f"oracle3_ask_window failed rc={rc}")
    return out, _stats_list(st, MAX_LEVELS)


def ask3_by_lookup(E: np.ndarray, g: int, r: int, B: int):
    """3-D ASK decisions replayed over an exhaustive volume E [z, y, x]."""
    E = np.ascontiguousarray(E, dtype=np.int32)
    n = E.shape[0]
    out = np.full((n, n, n), -1, dtype=np.int32)
    st = (LevelStats * MAX_LEVELS)()
    rc = lib().oracle3_ask_by_lookup(_i32(E), n, g, r, B, _i32(out), st, MAX_LEVELS)
    if rc != 0:
        raise ValueError(f"oracle3_ask_by_lookup failed rc={rc}")
    return out, _stats_list(st, MAX_LEVELS)
