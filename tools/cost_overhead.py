"""Device time of one ASK step under the multi-GPU plan's options (dev tool, GPU box): plain,
device tile list (all tiles, LPT order), and the sampled / exact per-tile cost counters; for
the full image and for the heaviest rank of an 8-way deal.

    python tools/cost_overhead.py [C3 ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_02255_b200 import multigpu  # noqa: E402


def ev(fn, flush, reps=7):
    fn()
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return round(statistics.median(ts), 4)


def main():
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for nm in sys.argv[1:] or ["C3"]:
        w = W.CONFIGS[nm]
        out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
        ws = mb.workspace(w.n, w.g, w.r, w.B)
        A = lambda **k: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, **k)  # noqa: E731
        res = {"w": nm, "plain": ev(lambda: A(), flush)}
        for P in (1, 8):
            plan = multigpu.DevicePlan(w, P, 0, torch.device("cuda"))
            mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tile_cost=True)
            costs = mb.tile_cost_view(ws, w.n, w.g, w.r, w.B).clone()
            plan.deal(costs, both=True)
            host = plan.host_tiles()
            d = (plan.tiles, plan.count)
            res[f"P{P}"] = {
                "host_tiles": ev(lambda: A(tiles=host), flush),
                "dtiles": ev(lambda: A(dtiles=d), flush),
                "dtiles_sampled": ev(lambda: A(dtiles=d, tile_cost="sampled"), flush),
                "dtiles_exact": ev(lambda: A(dtiles=d, tile_cost=True), flush),
                "canonical_sampled": ev(lambda: A(tiles=sorted(host), tile_cost="sampled"), flush),
                "canonical": ev(lambda: A(tiles=sorted(host)), flush),
            }
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
