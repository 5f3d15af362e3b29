"""ctypes binding of libmandel_b200.so (include/mandel.h) -- argument marshalling only.

Every step of the path runs in the library's sm_100a kernels; this module only converts
Python/torch arguments to the C ABI.  There is no CPU fallback: if the library is missing
or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import List, Optional, Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
# MANDEL_B200_LIB: alternative build of the same library (tuning sweeps build variants with
# different -D knobs into gpurun_out/); default: the in-tree build.
LIB_PATH = os.environ.get("MANDEL_B200_LIB") or os.path.join(HERE, "libmandel_b200.so")

MANDEL_OK, MANDEL_EINVAL, MANDEL_EWORKSPACE, MANDEL_ECUDA = 0, 1, 2, 3
SCHEME_SBR, SCHEME_B200, SCHEME_MBR = 0, 1, 2
FLAG_STATS = 1
FLAG_TIMING = 2
FLAG_TILE_COST = 4
FLAG_FLAT = 8
FLAG_SERIAL = 16
FLAG_TILE_COST_SAMPLED = 32
FLAG_TIMING_LEAF = 128
MAX_GROUPS = 8


def flag_groups(g: int) -> int:
    """MANDEL_FLAG_GROUPS(g) of include/mandel.h."""
    if not 1 <= int(g) <= MAX_GROUPS:
        raise ValueError(f"groups must be in [1, {MAX_GROUPS}]")
    return ((int(g) - 1) & 15) << 8
KIND_NAMES = {0: "init", 1: "b200_border", 2: "b200_classify", 3: "fill", 4: "b200_leaf",
              5: "sbr_level", 6: "sbr_leaf", 7: "mbr_leaf"}

_lock = threading.Lock()
_lib: Optional[ctypes.CDLL] = None


class MandelRegion(ctypes.Structure):
    _fields_ = [("re_min", ctypes.c_double), ("re_max", ctypes.c_double),
                ("im_min", ctypes.c_double), ("im_max", ctypes.c_double)]


class MandelLevelStats(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32), ("side", ctypes.c_int32)] + [
        (k, ctypes.c_int64) for k in ("regions_in", "filled", "subdivided", "leaves",
                                       "border_px", "border_iters", "leaf_px", "leaf_iters")]


class MandelError(RuntimeError):
    def __init__(self, code: int, what: str):
        lib = load()
        msg = lib.mandel_strerror(code).decode()
        if code == MANDEL_ECUDA:
            msg += ": " + lib.mandel_last_cuda_error().decode()
        super().__init__(f"{what}: {msg} (code {code})")
        self.code = code


# (name, restype, argtypes) of every exported symbol declared in include/mandel.h
_P = ctypes.c_void_p
_SIGS = [
    ("mandel_ask_workspace_bytes", ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    ("mandel_ask_levels", ctypes.c_int32, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    ("mandel_exhaustive", ctypes.c_int, [MandelRegion, ctypes.c_int64, ctypes.c_int32, _P, ctypes.c_int64, _P]),
    ("mandel_exhaustive_tuned", ctypes.c_int, [MandelRegion, ctypes.c_int64, ctypes.c_int32, _P, ctypes.c_int64, _P]),
    ("mandel_ask", ctypes.c_int, [MandelRegion, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                  ctypes.c_int32, _P, ctypes.c_int64, _P, ctypes.c_size_t, _P]),
    ("mandel_ask_tiles", ctypes.c_int, [MandelRegion, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_int32, _P, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, _P,
                                        ctypes.c_int64, _P, ctypes.c_size_t, _P]),
    ("mandel_ask_dtiles", ctypes.c_int, [MandelRegion, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, _P, _P, ctypes.c_int32, ctypes.c_uint32, _P,
                                         ctypes.c_int64, _P, ctypes.c_size_t, _P]),
    ("mandel_deal_lpt", ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P, _P]),
    ("mandel_ask_tile_costs_offset", ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                                       ctypes.c_int32]),
    ("mandel_ask_to_host", ctypes.c_int, [MandelRegion, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_int32, _P, ctypes.c_int32, ctypes.c_int32, _P,
                                          ctypes.c_int64, _P, ctypes.c_size_t, _P, _P]),
    ("mandel_ask_to_host_u16", ctypes.c_int, [MandelRegion, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.c_int32, _P, ctypes.c_int32, ctypes.c_int32,
                                              _P, ctypes.c_int64, _P, ctypes.c_size_t, _P, _P, _P]),
    ("mandel_ask_last_stats", ctypes.c_int, [_P, ctypes.POINTER(MandelLevelStats), ctypes.c_int32, _P]),
    ("mandel_ask_kernel_count", ctypes.c_int32, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                 ctypes.c_int32]),
    ("mandel_ask_graph_captures", ctypes.c_longlong, []),
    ("mandel_fp32_peak_probe", ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(ctypes.c_double), _P]),
    ("mandel_ask_kernel_times", ctypes.c_int, [_P, _P, ctypes.c_int32]),
    ("mandel_ask_tile_costs", ctypes.c_int, [_P, _P, ctypes.c_int32, _P]),
    ("mandel_strerror", ctypes.c_char_p, [ctypes.c_int]),
    ("mandel_last_cuda_error", ctypes.c_char_p, []),
    ("mandel_shutdown", None, []),
]
EXPORTED = [s[0] for s in _SIGS]


def load() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(the CUDA extension is required; there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, res, args in _SIGS:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


# ---------------------------------------------------------------- Dynamic Parallelism library
# libmandel_dp.so (include/mandel_dp.h): the paper's recursive DP baseline, built separately
# with relocatable device code.
DP_LIB_PATH = os.environ.get("MANDEL_DP_LIB") or os.path.join(HERE, "libmandel_dp.so")
_DP_SIGS = [
    ("mandel_dp_pending_launches", ctypes.c_int64, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    ("mandel_dp", ctypes.c_int, [MandelRegion, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                 ctypes.c_int32, _P, ctypes.c_int64, _P]),
    ("mandel_dp_last_cuda_error", ctypes.c_char_p, []),
]
DP_EXPORTED = [s[0] for s in _DP_SIGS]
_dp_lib: Optional[ctypes.CDLL] = None


def load_dp() -> ctypes.CDLL:
    global _dp_lib
    with _lock:
        if _dp_lib is None:
            if not os.path.exists(DP_LIB_PATH):
                raise RuntimeError(f"{DP_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                                   "g.build()'` (no CPU fallback)")
            lib = ctypes.CDLL(DP_LIB_PATH)
            for name, res, args in _DP_SIGS:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _dp_lib = lib
    return _dp_lib


def check_dp(code: int, what: str) -> None:
    if code != MANDEL_OK:
        msg = load().mandel_strerror(code).decode()
        if code == MANDEL_ECUDA:
            msg += ": " + load_dp().mandel_dp_last_cuda_error().decode()
        raise RuntimeError(f"{what}: {msg} (code {code})")


def region(r: Sequence[float]) -> MandelRegion:
    return MandelRegion(*[float(v) for v in r])


def check(code: int, what: str) -> None:
    if code != MANDEL_OK:
        raise MandelError(code, what)


def tiles_arg(tiles):
    if tiles is None:
        return None, 0, None
    arr = (ctypes.c_int32 * len(tiles))(*[int(t) for t in tiles])
    return ctypes.cast(arr, ctypes.c_void_p), len(tiles), arr


def stats(ws_ptr: int, stream_ptr: int, max_levels: int = 32) -> List[dict]:
    lib = load()
    buf = (MandelLevelStats * max_levels)()
    L = lib.mandel_ask_last_stats(ws_ptr, buf, max_levels, stream_ptr)
    if L < 0:
        raise MandelError(-L, "mandel_ask_last_stats")
    out = []
    for i in range(min(L, max_levels)):
        s = buf[i]
        out.append({k: int(getattr(s, k)) for k, _ in MandelLevelStats._fields_})
    return out


def kernel_times(max_kernels: int = 256) -> List[dict]:
    """Per-kernel device times of the last MANDEL_FLAG_TIMING call."""
    lib = load()
    ms = (ctypes.c_float * max_kernels)()
    kl = (ctypes.c_int32 * max_kernels)()
    nk = lib.mandel_ask_kernel_times(ctypes.cast(ms, ctypes.c_void_p), ctypes.cast(kl, ctypes.c_void_p),
                                     max_kernels)
    if nk < 0:
        raise MandelError(-nk, "mandel_ask_kernel_times")
    return [{"kind": KIND_NAMES[kl[i] // 100], "level": kl[i] % 100, "ms": float(ms[i])}
            for i in range(min(nk, max_kernels))]


def tile_costs(ws_ptr: int, g: int, stream_ptr: int) -> List[int]:
    lib = load()
    buf = (ctypes.c_uint64 * (g * g))()
    rc = lib.mandel_ask_tile_costs(ws_ptr, ctypes.cast(buf, ctypes.c_void_p), g * g, stream_ptr)
    if rc < 0:
        raise MandelError(-rc, "mandel_ask_tile_costs")
    return [int(v) for v in buf]


# ---------------------------------------------------------------- libmandel3d.so (k = 3)
LIB3_PATH = os.environ.get("MANDEL3D_LIB") or os.path.join(HERE, "libmandel3d.so")


class Mandel3dRegion(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("re_min", "re_max", "im_min", "im_max", "w_min", "w_max")]


class Mandel3dLevelStats(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32), ("side", ctypes.c_int32)] + [
        (k, ctypes.c_int64) for k in ("regions_in", "filled", "subdivided", "leaves",
                                       "border_px", "border_iters", "leaf_px", "leaf_iters")]


_SIGS3 = [
    ("mandel3d_ask_workspace_bytes", ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                                       ctypes.c_int32]),
    ("mandel3d_ask_levels", ctypes.c_int32, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    ("mandel3d_exhaustive", ctypes.c_int, [Mandel3dRegion, ctypes.c_int64, ctypes.c_int32, _P, _P]),
    ("mandel3d_ask", ctypes.c_int, [Mandel3dRegion, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                    ctypes.c_int32, ctypes.c_uint32, _P, _P, ctypes.c_size_t, _P]),
    ("mandel3d_ask_last_stats", ctypes.c_int, [_P, ctypes.POINTER(Mandel3dLevelStats), ctypes.c_int32, _P]),
    ("mandel3d_last_cuda_error", ctypes.c_char_p, []),
    ("mandel3d_shutdown", None, []),
]
EXPORTED3 = [s[0] for s in _SIGS3]
_lib3: Optional[ctypes.CDLL] = None


def load_3d() -> ctypes.CDLL:
    global _lib3
    with _lock:
        if _lib3 is None:
            if not os.path.exists(LIB3_PATH):
                raise RuntimeError(f"{LIB3_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                                   "g.build()'` (no CPU fallback)")
            lib = ctypes.CDLL(LIB3_PATH)
            for name, res, args in _SIGS3:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib3 = lib
    return _lib3


def check3(rc: int, what: str) -> None:
    if rc != 0:
        err = load_3d().mandel3d_last_cuda_error().decode()
        raise MandelError3(rc, f"{what}: code {rc} ({'invalid argument' if rc == 1 else 'workspace too small' if rc == 2 else err})")


class MandelError3(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
