"""Independent level chains (MANDEL_FLAG_GROUPS) at the heaviest rank's share of an 8-way LPT
deal and at the full image (dev tool, GPU box): device time per ASK step for G = 1, 2, 4.

    python tools/groups_rank.py [C3 ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_02255_b200 import deal  # noqa: E402


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
        mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tile_cost=True)
        exact = mb.tile_costs(ws, w.g)
        heavy = max(deal.deal("lpt", w.g, 8, exact), key=lambda p: sum(exact[k] for k in p))
        res = {"w": nm}
        for G in (1, 2, 3, 4):
            res[f"rank8_G{G}"] = ev(lambda: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws,
                                                   tiles=heavy, groups=G), flush)
            res[f"full_G{G}"] = ev(lambda: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws,
                                                  groups=G), flush)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
