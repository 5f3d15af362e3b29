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
# Frames between two sampled (counted) renders: the counters cost ~2.4% of a rank's step
# (tools/ab_variants.py C4r8d vs C4r8n), so only every third frame counts and re-deals; with
# two alternating tile lists and an odd period, each list is re-dealt every 2 * SAMPLE_EVERY
# frames.
SAMPLE_EVERY = 3


class DevicePlan:
    """One rank's device-resident level-0 deal for workload `w`.

    Two device tile lists (int32 cuda tensors, read by mandel_ask_dtiles when a step executes)
    alternate between steps.  deal(costs) overwrites the current one with this rank's share of
    an LPT schedule of the g*g per-tile costs (mandel_deal_lpt: identical on every rank for
    identical costs).  step() is the frame loop of bench.py: render with sampled per-tile cost
    counters, then -- on a side stream, overlapped with the NEXT step's render -- all-reduce
    the counters and deal the step after next (a one-step-lagged feedback plan, so the plan is
    off the critical path but still inside the timed region's wall time)."""

    def __init__(self, w, world: int, rank: int, device, shrink: int = PREVIEW_SHRINK,
                 dwell_shrink: int = PREVIEW_DWELL_SHRINK, sample_every: int = SAMPLE_EVERY):
        import torch
        from . import ask, workspace
        self.w, self.world, self.rank, self.device = w, world, rank, device
        G = w.g * w.g
        self.tiles2 = [torch.arange(G, dtype=torch.int32, device=device) for _ in range(2)]
        self.count2 = [torch.tensor([G], dtype=torch.int32, device=device) for _ in range(2)]
        self.cbuf2 = [torch.zeros(G, dtype=torch.int64, device=device) for _ in range(2)]
        self.cur = 0
        self.side = torch.cuda.Stream(device=device)
        self.ev_plan = [None, None]
        self.pn = max(2 * w.g, w.n // shrink)
        self.pB = max(2, w.B // shrink)
        while w.g * self.pB > self.pn:
            self.pB //= 2
        self.pmd = max(1, w.maxdwell // dwell_shrink)
        self.pws = workspace(self.pn, w.g, w.r, self.pB, device=device)
        self.pout = torch.empty((self.pn, self.pn), dtype=torch.int32, device=device)
        self._ask = ask
        self.sample_every = max(1, int(sample_every))
        self.n_steps = 0

    @property
    def tiles(self):
        return self.tiles2[self.cur]

    @property
    def count(self):
        return self.count2[self.cur]

    def preview_costs(self, costs_out):
        """Per-tile executed iterations of ASK on the n/shrink, maxdwell/dwell_shrink preview
        (the first steps' cost estimate), copied into the int64 tensor costs_out."""
        from . import tile_cost_view
        w = self.w
        self._ask(w.region, self.pn, self.pmd, w.g, w.r, self.pB, out=self.pout, ws=self.pws, tile_cost=True)
        costs_out.copy_(tile_cost_view(self.pws, self.pn, w.g, w.r, self.pB))

    def deal(self, costs, both: bool = False):
        """Deal the current tile list (both: both lists) on the current stream."""
        from . import deal_lpt
        for k in ((0, 1) if both else (self.cur,)):
            deal_lpt(costs, self.world, self.rank, self.tiles2[k], self.count2[k])

    def render(self, out, ws, tile_cost="sampled", timing=False):
        """This rank's ASK over its current tiles (device list), estimating per-tile work
        (MANDEL_FLAG_TILE_COST_SAMPLED) for a later step's deal."""
        w = self.w
        return self._ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws,
                         dtiles=(self.tiles, self.count), tile_cost=tile_cost, timing=timing)

    def step(self, out, ws, allreduce, timing=False):
        """One frame: wait for the plan that chose this step's tiles and render them.  Every
        `sample_every`-th frame renders with the sampled counters and hands them to the side
        stream, which all-reduces them (`allreduce(t)`: in place, sum over ranks) and deals the
        step after next into the list this step just used; the other frames render without
        counters and keep their list.  Every rank calls allreduce on the same frames."""
        import torch
        from . import deal_lpt, tile_cost_view
        w, k = self.w, self.cur
        main = torch.cuda.current_stream(self.device)
        if self.ev_plan[k] is not None:
            main.wait_event(self.ev_plan[k])
        sample = self.n_steps % self.sample_every == 0
        self.n_steps += 1
        if not sample:
            self.render(out, ws, tile_cost=False, timing=timing)
            self.cur = 1 - k
            return
        self.render(out, ws, timing=timing)
        cb = self.cbuf2[k]
        cb.copy_(tile_cost_view(ws, w.n, w.g, w.r, w.B))
        ev = torch.cuda.Event()
        ev.record(main)
        with torch.cuda.stream(self.side):
            self.side.wait_event(ev)
            allreduce(cb)
            deal_lpt(cb, self.world, self.rank, self.tiles2[k], self.count2[k], stream=self.side)
            ev_p = torch.cuda.Event()
            ev_p.record(self.side)
        self.ev_plan[k] = ev_p
        self.cur = 1 - k

    def host_tiles(self, which: int = None):
        """Tile list `which` (default: the next step's) on the host (synchronises)."""
        import torch
        k = self.cur if which is None else which
        torch.cuda.synchronize(self.device)
        return self.tiles2[k][: int(self.count2[k].item())].tolist()
