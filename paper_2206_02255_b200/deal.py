"""Multi-GPU partition of the level-0 regions (BASELINE.json config 3-5, north_star
"initial g x g regions are dealt cyclically across ranks").

Level-0 regions are independent (every ASK decision is local to a region), so
ranks never exchange data on the hot path: each runs mandel_ask_tiles on its own tiles.
Deals (tile id k = gy * g + gx, canonical order):
  cyclic     k -> rank k mod P                       (plain cyclic deal)
  diagonal   k -> rank (gx + gy) mod P               (balances conjugate mirror pairs)
  costrank   tiles sorted by an estimated cost (descending, ties by id), dealt
             boustrophedon 0..P-1, P-1..0, ...       (cost-ranked cyclic deal); each rank
             keeps its tiles in that descending order, which becomes its level-0 OLT order
             (longest-first: the level-0 kernel's tail is short work)
  lpt        the same cost order, each tile to the currently least-loaded rank (ties: lowest
             rank) -- Graham's longest-processing-time-first list schedule; balances better
             than boustrophedon when a few tiles dominate (the seahorse window, C5)
"""
from __future__ import annotations

from typing import List, Optional, Sequence


def cyclic(g: int, world: int) -> List[List[int]]:
    return [[k for k in range(g * g) if k % world == r] for r in range(world)]


def diagonal(g: int, world: int) -> List[List[int]]:
    return [[k for k in range(g * g) if ((k % g) + (k // g)) % world == r] for r in range(world)]


def costrank(costs: Sequence[float], world: int) -> List[List[int]]:
    order = sorted(range(len(costs)), key=lambda k: (-float(costs[k]), k))
    out: List[List[int]] = [[] for _ in range(world)]
    for i, k in enumerate(order):
        rnd, pos = divmod(i, world)
        out[pos if rnd % 2 == 0 else world - 1 - pos].append(k)
    return out  # each rank's tiles in descending cost: its level-0 work starts with the longest


def lpt(costs: Sequence[float], world: int) -> List[List[int]]:
    order = sorted(range(len(costs)), key=lambda k: (-float(costs[k]), k))
    out: List[List[int]] = [[] for _ in range(world)]
    load = [0.0] * world
    for k in order:
        r = min(range(world), key=lambda q: (load[q], q))
        out[r].append(k)
        load[r] += float(costs[k])
    return out  # descending cost within each rank, like costrank


def deal(method: str, g: int, world: int, costs: Optional[Sequence[float]] = None) -> List[List[int]]:
    if method == "cyclic":
        return cyclic(g, world)
    if method == "diagonal":
        return diagonal(g, world)
    if method == "costrank":
        if costs is None:
            raise ValueError("costrank needs per-tile costs")
        return costrank(costs, world)
    if method == "lpt":
        if costs is None:
            raise ValueError("lpt needs per-tile costs")
        return lpt(costs, world)
    raise ValueError(method)


def imbalance(parts: Sequence[Sequence[int]], costs: Sequence[float]) -> float:
    """max over ranks / mean over ranks of the summed tile costs."""
    loads = [sum(float(costs[k]) for k in p) for p in parts]
    mean = sum(loads) / len(loads)
    return max(loads) / mean if mean > 0 else 1.0
