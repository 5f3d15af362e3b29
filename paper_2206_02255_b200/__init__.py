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

SCHEMES = {"sbr": _lib.SCHEME_SBR, "b200": _lib.SCHEME_B200, "mbr": _lib.SCHEME_MBR}
# Independent ASK chains per call (MANDEL_FLAG_GROUPS); same image for any value.
DEFAULT_GROUPS = 1


def _torch():
    import torch
    return torch


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _check_device(out, *others, stream=None):
    """The library launches on the CURRENT device (cudaGetDevice): every buffer and the stream
    must live on out's device; the caller wraps the call in `torch.cuda.device(out.device)`."""
    for t in others:
        if t is not None and t.device != out.device:
            raise ValueError(f"buffer on {t.device} but out is on {out.device}")
    if stream is not None and stream.device != out.device:
        raise ValueError(f"stream on {stream.device} but out is on {out.device}")


def _temp_workspace(n, g, r, B, out, stream):
    """A call-local workspace: allocated on out's device, and tied to `stream` (record_stream)
    when that is not the current stream, so the caching allocator does not hand its memory to
    another allocation while the graph launched on `stream` still uses it."""
    torch = _torch()
    ws = workspace(n, g, r, B, device=out.device)
    if stream is not None and stream != torch.cuda.current_stream(out.device):
        ws.record_stream(stream)
    return ws


def levels(n: int, g: int, r: int, B: int) -> int:
    return int(_lib.load().mandel_ask_levels(n, g, r, B))


def workspace_bytes(n: int, g: int, r: int, B: int) -> int:
    v = int(_lib.load().mandel_ask_workspace_bytes(n, g, r, B))
    if v == 0:
        raise ValueError(f"invalid ASK parameters n={n} g={g} r={r} B={B}")
    return v


def kernel_count(n: int, g: int, r: int, B: int, scheme: str = "b200") -> int:
    """Kernel launches of one ask() call."""
    return int(_lib.load().mandel_ask_kernel_count(n, g, r, B, SCHEMES[scheme]))


def graph_captures() -> int:
    """CUDA graphs captured so far by the library (one per launch shape; regions, maxdwell and
    tile lists are per-call parameters and reuse it)."""
    return int(_lib.load().mandel_ask_graph_captures())


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


def exhaustive(region: Sequence[float], n: int, maxdwell: int, out=None, stream=None, tuned: bool = False):
    """Exhaustive dwell image: one thread per pixel.  tuned: the kernel with
    32-step escape-test chunks (mandel_exhaustive_tuned; same image)."""
    out = _image(n, out)
    _check_device(out, stream=stream)
    lib = _lib.load()
    fn = lib.mandel_exhaustive_tuned if tuned else lib.mandel_exhaustive
    with _torch().cuda.device(out.device):
        rc = fn(_lib.region(region), n, maxdwell, out.data_ptr(), out.stride(0), _stream_ptr(stream))
    _lib.check(rc, "mandel_exhaustive_tuned" if tuned else "mandel_exhaustive")
    return out


def dp(region: Sequence[float], n: int, maxdwell: int, g: int, r: int, B: int, out=None, stream=None):
    """The paper's Dynamic Parallelism baseline (include/mandel_dp.h, libmandel_dp.so):
    recursive Mariani-Silver, one child grid per subdividing node.  Same image as ask()."""
    out = _image(n, out)
    _check_device(out, stream=stream)
    with _torch().cuda.device(out.device):
        rc = _lib.load_dp().mandel_dp(_lib.region(region), n, maxdwell, g, r, B, out.data_ptr(), out.stride(0),
                                      _stream_ptr(stream))
    _lib.check_dp(rc, "mandel_dp")
    return out


def ask(region: Sequence[float], n: int, maxdwell: int, g: int, r: int, B: int, out=None, ws=None,
        tiles: Optional[Sequence[int]] = None, scheme: str = "b200", stats: bool = False,
        timing: bool = False, tile_cost: bool = False, flat: bool = False, serial: bool = False,
        groups: Optional[int] = None, stream=None, dtiles=None):
    """ASK dwell image over all g*g level-0 regions, or only `tiles`.
    stats: accumulate per-level counters (ask_stats); timing: per-kernel events
    (kernel_times; "leaf": around the leaf kernel only, which keeps the level chain's
    programmatic-dependent-launch edges); flat: B200 scheme with the plain thread-per-pixel
    border/leaf kernels instead of the lane-refill ones; serial: fills on the main stream
    instead of concurrent graph branches (A/B comparisons, same image); groups: independent
    level-synchronous chains over round-robin subsets of the tiles, run as parallel graph
    branches.  tile_cost: True counts every level-0 tile's executed iterations exactly;
    "sampled" estimates a time proxy from the 1/64 pixel lattice (x + y) % 64 == 0, each
    sampled pixel counted as 64 * (dwell + 64): iterations plus the per-pixel work (B200
    scheme; the multi-GPU deal's per-step feedback)."""
    out = _image(n, out)
    _check_device(out, ws, stream=stream)
    if ws is None:
        ws = _temp_workspace(n, g, r, B, out, stream)
    t_ptr, t_n, _keep = _lib.tiles_arg(tiles)
    flags = ((_lib.FLAG_STATS if stats else 0)
             | (_lib.FLAG_TIMING_LEAF if timing == "leaf" else _lib.FLAG_TIMING if timing else 0)
             | (_lib.FLAG_TILE_COST_SAMPLED if tile_cost == "sampled" else _lib.FLAG_TILE_COST if tile_cost else 0)
             | (_lib.FLAG_FLAT if flat else 0)
             | (_lib.FLAG_SERIAL if serial else 0)
             | _lib.flag_groups(DEFAULT_GROUPS if groups is None else groups))
    with _torch().cuda.device(out.device):
        if dtiles is not None:
            rc = _lib.load().mandel_ask_dtiles(_lib.region(region), n, maxdwell, g, r, B, dtiles[0].data_ptr(),
                                               dtiles[1].data_ptr(), SCHEMES[scheme], flags, out.data_ptr(),
                                               out.stride(0), ws.data_ptr(), ws.numel(), _stream_ptr(stream))
        else:
            rc = _lib.load().mandel_ask_tiles(_lib.region(region), n, maxdwell, g, r, B, t_ptr, t_n,
                                              SCHEMES[scheme], flags, out.data_ptr(), out.stride(0),
                                              ws.data_ptr(), ws.numel(), _stream_ptr(stream))
    _lib.check(rc, "mandel_ask_dtiles" if dtiles is not None else "mandel_ask_tiles")
    return out


def tile_cost_view(ws, n: int, g: int, r: int, B: int):
    """The workspace's per-tile cost counters (MANDEL_FLAG_TILE_COST) as an int64 cuda tensor
    of g*g entries, a view into ws (for an in-place all-reduce across ranks)."""
    torch = _torch()
    off = int(_lib.load().mandel_ask_tile_costs_offset(n, g, r, B))
    if off == 0 or off % 8:
        raise ValueError("invalid ASK parameters")
    return ws[off:off + 8 * g * g].view(torch.int64)


def deal_lpt(costs, world: int, rank: int, tiles_out, count_out, stream=None):
    """Device-side LPT deal (mandel_deal_lpt): rank `rank`'s tiles of a `world`-way
    longest-processing-time schedule on the int64 cuda tensor `costs` (g*g, canonical order),
    written to the int32 cuda tensors tiles_out (>= g*g) and count_out (1), asynchronously."""
    torch = _torch()
    if costs.dtype != torch.int64 or tiles_out.dtype != torch.int32 or count_out.dtype != torch.int32:
        raise ValueError("deal_lpt: int64 costs, int32 outputs")
    _check_device(costs, tiles_out, count_out, stream=stream)
    with torch.cuda.device(costs.device):
        rc = _lib.load().mandel_deal_lpt(costs.data_ptr(), costs.numel(), world, rank, tiles_out.data_ptr(),
                                         count_out.data_ptr(), _stream_ptr(stream))
    _lib.check(rc, "mandel_deal_lpt")


def ask_stats(ws, stream=None) -> List[dict]:
    """Per-level statistics of the last ASK call on `ws` (synchronises the stream)."""
    with _torch().cuda.device(ws.device):
        return _lib.stats(ws.data_ptr(), _stream_ptr(stream))


def ask_to_host(region, n, maxdwell, g, r, B, h_out, out, ws, tiles=None, scheme="b200", stream=None,
                stage=None):
    """ASK through the C ABI into HOST memory h_out (n x n, ideally pinned).  h_out int32:
    mandel_ask_to_host.  h_out uint16 (or int16 holding the same bits): mandel_ask_to_host_u16,
    which narrows each finished band on the device into `stage` (n*n 16-bit device tensor,
    allocated here if None) and copies half the bytes; needs maxdwell <= 65535."""
    torch = _torch()
    u16 = h_out.dtype in (torch.uint16, torch.int16)
    if (h_out.dtype != torch.int32 and not u16) or h_out.is_cuda or not h_out.is_contiguous() \
            or h_out.numel() < n * n:
        raise ValueError("h_out must be a contiguous host int32 or uint16 tensor of n*n elements")
    _check_device(out, ws, stage, stream=stream)
    t_ptr, t_n, _keep = _lib.tiles_arg(tiles)
    with torch.cuda.device(out.device):
        if u16:
            if stage is None:
                stage = torch.empty(n * n, dtype=torch.int16, device=out.device)
                if stream is not None and stream != torch.cuda.current_stream():
                    stage.record_stream(stream)
            elif stage.dtype not in (torch.uint16, torch.int16) or stage.numel() < n * n \
                    or not stage.is_contiguous():
                raise ValueError("stage must be a contiguous 16-bit device tensor of n*n elements")
            rc = _lib.load().mandel_ask_to_host_u16(_lib.region(region), n, maxdwell, g, r, B, t_ptr, t_n,
                                                    SCHEMES[scheme], out.data_ptr(), out.stride(0), ws.data_ptr(),
                                                    ws.numel(), stage.data_ptr(), h_out.data_ptr(),
                                                    _stream_ptr(stream))
            _lib.check(rc, "mandel_ask_to_host_u16")
            return h_out
        rc = _lib.load().mandel_ask_to_host(_lib.region(region), n, maxdwell, g, r, B, t_ptr, t_n,
                                            SCHEMES[scheme], out.data_ptr(), out.stride(0), ws.data_ptr(),
                                            ws.numel(), h_out.data_ptr(), _stream_ptr(stream))
    _lib.check(rc, "mandel_ask_to_host")
    return h_out


def tile_costs(ws, g: int, stream=None) -> List[int]:
    """Executed iterations per level-0 tile of the last ask(..., tile_cost=True) on `ws`."""
    with _torch().cuda.device(ws.device):
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


def fp32_peak_tops(steps: int = 2048, stream=None) -> float:
    """Measured FP32 rate of the dwell step on the current device, T ops/s (ALU roofline
    denominator; mandel_fp32_peak_probe)."""
    import ctypes
    v = ctypes.c_double(0.0)
    _lib.check(_lib.load().mandel_fp32_peak_probe(steps, ctypes.byref(v), _stream_ptr(stream)),
               "mandel_fp32_peak_probe")
    return float(v.value)


def kernel_times() -> List[dict]:
    """Per-kernel device times (ms) of the most recent ask(..., timing=True) call."""
    return _lib.kernel_times()


def shutdown() -> None:
    _lib.load().mandel_shutdown()
