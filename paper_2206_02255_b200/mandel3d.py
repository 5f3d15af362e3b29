"""ASK on k = 3 orthotopes (NEXT-4; the paper's Sec. 6.2): the
(c_re, c_im, w) dwell volume with z_0 = w, subdivided by surface tests.  Every computation
runs in libmandel3d.so's sm_100a kernels through the C ABI of include/mandel3d.h; torch only
supplies device memory and the stream.

    exhaustive3d(region3, n, maxdwell, out=None)                 -> int32 (n, n, n) [z, y, x]
    ask3d(region3, n, maxdwell, g, r, B, out=None, ws=None, stats=False) -> same shape
    ask3d_stats(ws)                                              -> per-level dict list
"""
from __future__ import annotations

from typing import List, Sequence

from . import _lib

MAX_LEVELS = 16


def _torch():
    import torch
    return torch


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _check_device(out, *others, stream=None):
    """libmandel3d.so launches on the current device: buffers and stream must be on out's."""
    for t in others:
        if t is not None and t.device != out.device:
            raise ValueError(f"buffer on {t.device} but out is on {out.device}")
    if stream is not None and stream.device != out.device:
        raise ValueError(f"stream on {stream.device} but out is on {out.device}")


def levels3d(n: int, g: int, r: int, B: int) -> int:
    return int(_lib.load_3d().mandel3d_ask_levels(n, g, r, B))


def workspace3d(n: int, g: int, r: int, B: int, device=None):
    torch = _torch()
    v = int(_lib.load_3d().mandel3d_ask_workspace_bytes(n, g, r, B))
    if v == 0:
        raise ValueError(f"invalid 3-D ASK parameters n={n} g={g} r={r} B={B}")
    return torch.empty(v, dtype=torch.uint8, device=device if device is not None else "cuda")


def _volume(n: int, out, device=None):
    torch = _torch()
    if out is None:
        out = torch.empty((n, n, n), dtype=torch.int32, device=device if device is not None else "cuda")
    if out.dtype != torch.int32 or tuple(out.shape) != (n, n, n) or not out.is_contiguous() or not out.is_cuda:
        raise ValueError("out must be a contiguous cuda int32 (n, n, n) tensor")
    return out


def _region(region3: Sequence[float]):
    return _lib.Mandel3dRegion(*[float(v) for v in region3])


def exhaustive3d(region3, n: int, maxdwell: int, out=None, stream=None):
    """Exhaustive dwell volume: one thread per voxel."""
    out = _volume(n, out)
    _check_device(out, stream=stream)
    with _torch().cuda.device(out.device):
        rc = _lib.load_3d().mandel3d_exhaustive(_region(region3), n, maxdwell, out.data_ptr(), _stream_ptr(stream))
    _lib.check3(rc, "mandel3d_exhaustive")
    return out


def ask3d(region3, n: int, maxdwell: int, g: int, r: int, B: int, out=None, ws=None, stats: bool = False,
          flat: bool = False, stream=None):
    """3-D ASK volume over all g^3 level-0 cubes (surface test, fill / r^3 split / leaf);
    flat: thread-per-voxel surface/leaf kernels instead of the lane-refill engine (A/B)."""
    out = _volume(n, out)
    _check_device(out, ws, stream=stream)
    if ws is None:
        ws = workspace3d(n, g, r, B, device=out.device)
        torch = _torch()
        if stream is not None and stream != torch.cuda.current_stream(out.device):
            ws.record_stream(stream)  # a call-local workspace must outlive the launch on `stream`
    with _torch().cuda.device(out.device):
        rc = _lib.load_3d().mandel3d_ask(_region(region3), n, maxdwell, g, r, B,
                                         (1 if stats else 0) | (2 if flat else 0), out.data_ptr(),
                                         ws.data_ptr(), ws.numel(), _stream_ptr(stream))
    _lib.check3(rc, "mandel3d_ask")
    return out


def ask3d_stats(ws, stream=None) -> List[dict]:
    buf = (_lib.Mandel3dLevelStats * MAX_LEVELS)()
    with _torch().cuda.device(ws.device):
        L = _lib.load_3d().mandel3d_ask_last_stats(ws.data_ptr(), buf, MAX_LEVELS, _stream_ptr(stream))
    if L < 0:
        raise RuntimeError("mandel3d_ask_last_stats failed")
    return [{k: int(getattr(buf[i], k)) for k, _ in _lib.Mandel3dLevelStats._fields_} for i in range(min(L, MAX_LEVELS))]
