"""B200-native ASK Mandelbrot (arxiv 2206.02255): the paper's Adaptive Serial Kernels
subdivision of the Mandelbrot dwell image, plus the exhaustive baseline, on sm_100a.

Python API (torch supplies device memory and streams; every computation runs in
libmandel_b200.so's CUDA kernels through the C ABI of include/mandel.h):

    exhaustive(region, n, maxdwell, out=None)                  -> int32 (n, n) cuda tensor
    ask(region, n, maxdwell, g, r, B, out=None, ws=None, tiles=None,
        scheme="b200", stats=False)                             -> int32 (n, n) cuda tensor
    ask_stats(ws)                                               -> per-level dict list
    ask_to_host(region, n, maxdwell, g, r, B, h_out, out, ws)   -> h_out (pinned host)
    workspace(n, g, r, B)                                       -> uint8 cuda tensor
    dp(region, n, maxdwell, g, r, B, out=None)                  -> int32 (n, n) cuda tensor
                                       (Dynamic Parallelism baseline, libmandel_dp.so)
"""
from __future__ import annotations

from typing import List, Optional, Sequence

from . import _lib

SCHEMES = {"sbr": _lib.SCHEME_SBR, "b200": _lib.SCHEME_B200, "mbr": _lib.SCHEME_MBR, "flow": _lib.SCHEME_FLOW}
# Independent ASK chains per call (MANDEL_FLAG_GROUPS); same image for any value.
DEFAULT_GROUPS = 1
# Deferred long pixels (MANDEL_FLAG_DEFER); same image either way.
DEFAULT_DEFER = False


def _torch():
    import torch
    return torch


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def levels(n: int, g: int, r: int, B: int) -> int:
    return int(_lib.load().mandel_ask_levels(n, g, r, B))


def workspace_bytes(n: int, g: int, r: int, B: int) -> int:
    v = int(_lib.load().mandel_ask_workspace_bytes(n, g, r, B))
    if v == 0:
        raise ValueError(f"invalid ASK parameters n={n} g={g} r={r} B={B}")
    return v


def kernel_count(n: int, g: int, r: int, B: int, scheme: str = "b200", defer=None, maxdwell: int = 0) -> int:
    """Kernel launches of one ask() call (defer / maxdwell as passed to ask())."""
    if not _lib.flag_defer(DEFAULT_DEFER if defer is None else defer):
        return int(_lib.load().mandel_ask_kernel_count(n, g, r, B, SCHEMES[scheme]))
    return int(_lib.load().mandel_ask_kernel_count_ex(n, g, r, B, SCHEMES[scheme],
                                                      _lib.flag_defer(DEFAULT_DEFER if defer is None else defer),
                                                      max(1, int(maxdwell))))


def workspace(n: int, g: int, r: int, B: int, device=None):
    torch = _torch()
    return torch.empty(workspace_bytes(n, g, r, B), dtype=torch.uint8,
                       device=device if device is not None else "cuda")


def _image(n: int, out, device=None):
    torch = _torch()
    if out is None:
        out = torch.empty((n, n), dtype=torch.int32, device=device if device is not None else "cuda")
    if out.dtype != torch.int32 or out.dim() != 2 or out.shape[0] < n or out.shape[1] < n \
            or out.stride(1) != 1 or not out.is_cuda:
        raise ValueError("out must be a cuda int32 (>=n, >=n) tensor with unit column stride")
    return out


def exhaustive(region: Sequence[float], n: int, maxdwell: int, out=None, stream=None):
    """Exhaustive dwell image: one thread per pixel."""
    out = _image(n, out)
    rc = _lib.load().mandel_exhaustive(_lib.region(region), n, maxdwell, out.data_ptr(),
                                       out.stride(0), _stream_ptr(stream))
    _lib.check(rc, "mandel_exhaustive")
    return out


def dp(region: Sequence[float], n: int, maxdwell: int, g: int, r: int, B: int, out=None, stream=None):
    """The paper's Dynamic Parallelism baseline (include/mandel_dp.h, libmandel_dp.so):
    recursive Mariani-Silver, one child grid per subdividing node.  Same image as ask()."""
    out = _image(n, out)
    rc = _lib.load_dp().mandel_dp(_lib.region(region), n, maxdwell, g, r, B, out.data_ptr(), out.stride(0),
                                  _stream_ptr(stream))
    _lib.check_dp(rc, "mandel_dp")
    return out


def ask(region: Sequence[float], n: int, maxdwell: int, g: int, r: int, B: int, out=None, ws=None,
        tiles: Optional[Sequence[int]] = None, scheme: str = "b200", stats: bool = False,
        timing: bool = False, tile_cost: bool = False, flat: bool = False, serial: bool = False,
        groups: Optional[int] = None, defer=None, stream=None):
    """ASK dwell image over all g*g level-0 regions, or only `tiles`.
    stats: accumulate per-level counters (ask_stats); timing: per-kernel events
    (kernel_times; "leaf": around the leaf kernel only, which keeps the level chain's
    programmatic-dependent-launch edges); flat: B200 scheme with the plain thread-per-pixel border/leaf kernels
    instead of the lane-refill ones; serial: fills on the main stream instead of concurrent
    graph branches (A/B comparisons, same image); groups: independent level-synchronous
    chains over round-robin subsets of the tiles, run as parallel graph branches; defer:
    MANDEL_FLAG_DEFER (True: default cap, int: that iteration cap, False: off)."""
    out = _image(n, out)
    if ws is None:
        ws = workspace(n, g, r, B, device=out.device)
    t_ptr, t_n, _keep = _lib.tiles_arg(tiles)
    rc = _lib.load().mandel_ask_tiles(_lib.region(region), n, maxdwell, g, r, B, t_ptr, t_n,
                                      SCHEMES[scheme],
                                      (_lib.FLAG_STATS if stats else 0)
                                      | (_lib.FLAG_TIMING_LEAF if timing == "leaf" else _lib.FLAG_TIMING if timing else 0)
                                      | (_lib.FLAG_TILE_COST if tile_cost else 0)
                                      | (_lib.FLAG_FLAT if flat else 0)
                                      | (_lib.FLAG_SERIAL if serial else 0)
                                      | _lib.flag_groups(DEFAULT_GROUPS if groups is None else groups)
                                      | _lib.flag_defer(DEFAULT_DEFER if defer is None else defer),
                                      out.data_ptr(), out.stride(0), ws.data_ptr(), ws.numel(),
                                      _stream_ptr(stream))
    _lib.check(rc, "mandel_ask_tiles")
    return out


def ask_stats(ws, stream=None) -> List[dict]:
    """Per-level statistics of the last ASK call on `ws` (synchronises the stream)."""
    return _lib.stats(ws.data_ptr(), _stream_ptr(stream))


def ask_to_host(region, n, maxdwell, g, r, B, h_out, out, ws, tiles=None, scheme="b200", stream=None):
    """ASK through the C ABI into HOST memory h_out (n x n int32, ideally pinned)."""
    torch = _torch()
    if h_out.dtype != torch.int32 or h_out.is_cuda or not h_out.is_contiguous() or h_out.numel() < n * n:
        raise ValueError("h_out must be a contiguous host int32 tensor of n*n elements")
    t_ptr, t_n, _keep = _lib.tiles_arg(tiles)
    rc = _lib.load().mandel_ask_to_host(_lib.region(region), n, maxdwell, g, r, B, t_ptr, t_n,
                                        SCHEMES[scheme], out.data_ptr(), out.stride(0), ws.data_ptr(),
                                        ws.numel(), h_out.data_ptr(), _stream_ptr(stream))
    _lib.check(rc, "mandel_ask_to_host")
    return h_out


def tile_costs(ws, g: int, stream=None) -> List[int]:
    """Executed iterations per level-0 tile of the last ask(..., tile_cost=True) on `ws`."""
    return _lib.tile_costs(ws.data_ptr(), g, _stream_ptr(stream))


def preview_costs(region, n: int, maxdwell: int, g: int, r: int, B: int, shrink: int = 8,
                  dwell_shrink: int = 2, scheme: str = "b200") -> List[int]:
    """Per-tile cost estimate for the cost-ranked deals: ASK itself on an
    n/shrink preview with maxdwell/dwell_shrink and B/shrink (>= 2), same g and r.  Default
    n/8, maxdwell/2: on the seahorse window (C5) the survey's n/16, maxdwell/8 preview misranks
    the dwell-heavy tiles (8-way imbalance 1.21-1.31 in executed iterations vs 1.02-1.06;
    profiles/r01_deals_*.jsonl)."""
    pn = max(g * 2, n // shrink)
    pB = max(2, B // shrink)
    while g * pB > pn:
        pB //= 2
    pmd = max(1, maxdwell // dwell_shrink)
    ws = workspace(pn, g, r, pB)
    ask(region, pn, pmd, g, r, pB, ws=ws, scheme=scheme, tile_cost=True)
    return tile_costs(ws, g)


def kernel_times() -> List[dict]:
    """Per-kernel device times (ms) of the most recent ask(..., timing=True) call."""
    return _lib.kernel_times()


def shutdown() -> None:
    _lib.load().mandel_shutdown()
