"""N > 1 host logic on CPU (gloo, world size 2): the level-0 tile deal, MAX/SUM reductions
and the verification gather of paper_2206_02255_b200.multigpu.  Each rank's tile image comes
from the oracle (CPU), so the data path of the CUDA kernels is not involved here; the GPU
parity tests cover mandel_ask_tiles itself."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W
from paper_2206_02255_b200 import deal, multigpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("method", ["cyclic", "diagonal", "costrank", "lpt"])
@pytest.mark.parametrize("g,world", [(16, 2), (16, 8), (4, 3), (8, 8), (2, 8)])
def test_deal_partitions(method, g, world):
    rng = np.random.default_rng(W.SEED)
    costs = rng.pareto(1.5, g * g).tolist() if method in ("costrank", "lpt") else None
    parts = deal.deal(method, g, world, costs)
    assert len(parts) == world
    flat = sorted(k for p in parts for k in p)
    assert flat == list(range(g * g))                       # disjoint and complete
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1 or method in ("diagonal", "lpt")


def test_costrank_balances_skewed_costs():
    # the survey's point: column-striped cyclic dealing is unbalanced on a
    # tile-cost map with a heavy column; cost-ranked boustrophedon dealing is not.
    g, world = 16, 8
    costs = np.ones((g, g))
    costs[:, 5] = 40.0
    costs = costs.ravel().tolist()
    cyc = deal.imbalance(deal.cyclic(g, world), costs)
    cr = deal.imbalance(deal.costrank(costs, world), costs)
    assert cyc > 2.0 and cr < 1.1


def test_lpt_list_schedule():
    """Graham's LPT list schedule (tiles in descending cost, each to the least-loaded rank,
    ties to the lowest rank), hand-traced on small cases, and never worse than the
    boustrophedon deal on a heavy-tailed seeded cost map."""
    assert deal.lpt([10, 6, 5, 5], 2) == [[0, 3], [1, 2]]
    # 8 -> r0; 7 -> r1; 6 -> r1 (7 < 8); 5 -> r0 (8 < 13); 4 -> r0 (13 == 13: lowest rank)
    assert deal.lpt([8, 7, 6, 5, 4], 2) == [[0, 3, 4], [1, 2]]
    # one dominant tile: it sits alone, the rest fill the other ranks
    parts = deal.lpt([100, 1, 1, 1, 1, 1, 1, 1, 1], 3)
    assert parts[0] == [0] and sorted(parts[1] + parts[2]) == list(range(1, 9))
    rng = np.random.default_rng(W.SEED + 3)
    costs = (rng.pareto(1.2, 256) + 1).tolist()
    assert deal.imbalance(deal.lpt(costs, 8), costs) <= deal.imbalance(deal.costrank(costs, 8), costs) + 1e-12


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, md, g, r, B = 256, 400, 8, 2, 8
        region = W.SEAHORSE_REGION
        # every rank must derive the same deal: identical (synthetic) per-tile costs
        costs = [float(k % 7 + 1) for k in range(g * g)]
        parts = deal.deal("costrank", g, world, costs)
        mine = multigpu.rank_tiles("costrank", g, world, rank, costs)
        assert mine == parts[rank]
        img, _ = oracle.ask(region, n, md, g, r, B, tiles=mine)
        full = multigpu.gather_image(torch.from_numpy(img), parts, g, rank)
        tmax = multigpu.max_over_ranks(10.0 + rank)
        tsum = multigpu.sum_over_ranks([1.0, float(rank)])
        if rank == 0:
            ref, _ = oracle.ask(region, n, md, g, r, B)
            q.put(("ok", bool(np.array_equal(full.numpy(), ref)), tmax, tsum))
        else:
            q.put(("ok", full is None, tmax, tsum))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_gather_and_reductions_world(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for status, ok, tmax, tsum in res:
        assert status == "ok", ok
        assert ok is True
        assert tmax == 10.0 + world - 1
        assert tsum == [float(world), float(sum(range(world)))]


def _worker_feedback(rank, world, port, q):
    """The host-visible logic of bench.py's N > 1 frame loop on gloo: every rank renders its
    tiles (oracle, per tile), reports their executed iterations in a g*g vector, all-reduces it,
    and re-deals with LPT for the frame after next (DevicePlan.step's one-step lag: the deal of
    frame f + 2 overlaps frame f + 1); all ranks must derive the same partition, the partition
    must be complete, and the gathered image must equal the single-process image."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, md, g, r, B = 256, 500, 8, 2, 8
        region = W.NONDYADIC_REGIONS[0]
        plans = [deal.diagonal(g, world), deal.cyclic(g, world)]  # frames 0, 1: static deals
        for frame in range(4):
            parts = plans[frame]
            mine = parts[rank]
            img = np.full((n, n), -1, np.int32)
            costs = torch.zeros(g * g, dtype=torch.int64)
            d0 = n // g
            for t in mine:
                tile, st = oracle.ask_tile(region, n, md, g, r, B, t)
                gy, gx = divmod(t, g)
                img[gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0] = tile
                costs[t] = sum(s["border_iters"] + s["leaf_iters"] for s in st)
            full = multigpu.gather_image(torch.from_numpy(img), parts, g, rank)
            dist.all_reduce(costs, op=dist.ReduceOp.SUM)
            nxt = deal.lpt(costs.tolist(), world)
            allp = [None] * world
            dist.all_gather_object(allp, nxt)
            assert all(p == nxt for p in allp)                       # same deal on every rank
            assert sorted(k for p in nxt for k in p) == list(range(g * g))
            if rank == 0:
                ref, _ = oracle.ask(region, n, md, g, r, B)
                assert np.array_equal(full.numpy(), ref), frame
            plans.append(nxt)  # frame + 2's deal
        parts = plans[-1]
        q.put(("ok", True, deal.imbalance(parts, costs.tolist()), None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_feedback_deal_world(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_feedback, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for status, ok, imb, _ in res:
        assert status == "ok", ok
        assert imb < 1.25
