"""Multi-GPU plumbing of the ASK path (north_star "Multi-GPU partition").

Level-0 regions are independent -- every ASK decision is local to a region --
so each rank runs mandel_ask_tiles on its own tiles and the hot path has no collective.
This module holds the host-side logic around it, written against torch.distributed so the
same code runs over NCCL on the GPU box and over gloo in the CPU tests:

  rank_tiles(...)        the rank's level-0 tiles under a deal (deal.py)
  max_over_ranks(v)      all_reduce(MAX) of a float (device-timed step totals)
  sum_over_ranks(vs)     all_reduce(SUM) of counters
  gather_image(...)      verification only: every rank packs its tiles into one contiguous
                         buffer, rank 0 receives them (batched point-to-point; NCCL over
                         NVLink on the box) and unpacks them into the full n x n image.
  DevicePlan             one rank's device-resident deal (tile list + count in device memory,
                         read by mandel_ask_dtiles when the step runs): first from an n/32,
                         maxdwell/8 preview, then every step from the previous step's per-tile
                         cost counters, all-reduced across ranks, through mandel_deal_lpt --
                         no host round trip between the plan and the rank's ASK.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

from . import deal as deal_mod


def _dist():
    import torch.distributed as dist
    return dist


def rank_tiles(method: str, g: int, world: int, rank: int,
               costs: Optional[Sequence[float]] = None) -> List[int]:
    parts = deal_mod.deal(method, g, world, costs)
    return parts[rank]


def max_over_ranks(value: float, device=None) -> float:
    import torch
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(values: Sequence[float], device=None) -> List[float]:
    import torch
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]


def pack_tiles(img, tiles: Sequence[int], g: int):
    """Contiguous (len(tiles), d0, d0) copy of the listed tiles of the n x n image `img`."""
    import torch
    n = img.shape[0]
    d0 = n // g
    out = torch.empty((len(tiles), d0, d0), dtype=img.dtype, device=img.device)
    for i, k in enumerate(tiles):
        gy, gx = divmod(int(k), g)
        out[i].copy_(img[gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0])
    return out


def unpack_tiles(img, packed, tiles: Sequence[int], g: int) -> None:
    n = img.shape[0]
    d0 = n // g
    for i, k in enumerate(tiles):
        gy, gx = divmod(int(k), g)
        img[gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0].copy_(packed[i])


def gather_image(img, parts: Sequence[Sequence[int]], g: int, rank: int, dst: int = 0):
    """Assemble the full image on rank `dst` from every rank's tiles (verification only, not
    on the timed path).  `parts[r]` are rank r's tiles; `img` is this rank's n x n buffer
    (only its own tiles are meaningful).  Returns the assembled image on dst, None elsewhere."""
    import torch
    dist = _dist()
    world = len(parts)
    mine = pack_tiles(img, parts[rank], g)
    if world == 1:
        return img
    if rank != dst:
        if len(parts[rank]):
            dist.send(mine.reshape(-1), dst)
        return None
    full = img
    unpack_tiles(full, mine, parts[rank], g)
    d0 = img.shape[0] // g
    bufs, ops = {}, []
    for r in range(world):
        if r == dst or not len(parts[r]):
            continue
        bufs[r] = torch.empty(len(parts[r]) * d0 * d0, dtype=img.dtype, device=img.device)
        ops.append(dist.P2POp(dist.irecv, bufs[r], r))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for r, b in bufs.items():
        unpack_tiles(full, b.reshape(len(parts[r]), d0, d0), parts[r], g)
    return full


PREVIEW_SHRINK, PREVIEW_DWELL_SHRINK = 32, 8  # n/32, maxdwell/8 (profiles/r02_preview_study.jsonl)


class DevicePlan:
    """One rank's device-resident level-0 deal for workload `w`.

    tiles / count are int32 cuda tensors that mandel_ask_dtiles reads when a step executes;
    deal(costs) overwrites them on the stream with this rank's share of an LPT schedule of the
    g*g per-tile costs (mandel_deal_lpt: identical on every rank for identical costs)."""

    def __init__(self, w, world: int, rank: int, device, shrink: int = PREVIEW_SHRINK,
                 dwell_shrink: int = PREVIEW_DWELL_SHRINK):
        import torch
        from . import ask, workspace
        self.w, self.world, self.rank, self.device = w, world, rank, device
        G = w.g * w.g
        self.tiles = torch.arange(G, dtype=torch.int32, device=device)
        self.count = torch.tensor([G], dtype=torch.int32, device=device)
        self.pn = max(2 * w.g, w.n // shrink)
        self.pB = max(2, w.B // shrink)
        while w.g * self.pB > self.pn:
            self.pB //= 2
        self.pmd = max(1, w.maxdwell // dwell_shrink)
        self.pws = workspace(self.pn, w.g, w.r, self.pB, device=device)
        self.pout = torch.empty((self.pn, self.pn), dtype=torch.int32, device=device)
        self._ask = ask

    def preview_costs(self, costs_out):
        """Per-tile executed iterations of ASK on the n/shrink, maxdwell/dwell_shrink preview
        (the first step's cost estimate), copied into the int64 tensor costs_out."""
        from . import tile_cost_view
        w = self.w
        self._ask(w.region, self.pn, self.pmd, w.g, w.r, self.pB, out=self.pout, ws=self.pws, tile_cost=True)
        costs_out.copy_(tile_cost_view(self.pws, self.pn, w.g, w.r, self.pB))

    def deal(self, costs):
        from . import deal_lpt
        deal_lpt(costs, self.world, self.rank, self.tiles, self.count)

    def render(self, out, ws, tile_cost: bool = True, timing=False):
        """This rank's ASK over its current tiles (device list), counting per-tile work."""
        w = self.w
        return self._ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws,
                         dtiles=(self.tiles, self.count), tile_cost=tile_cost, timing=timing)

    def host_tiles(self):
        """This rank's current tile list on the host (synchronises; verification only)."""
        return self.tiles[: int(self.count.item())].tolist()
