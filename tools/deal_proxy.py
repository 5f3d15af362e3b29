"""Which per-tile cost balances the 8-way deal in TIME (dev tool, GPU box)?

    python tools/deal_proxy.py [C3 C4 C5] [--P 8] [--reps 3]

Per-tile statistics come from the oracle's committed records (tests/golden/oracle_tiles: the
exact border/leaf pixels and iterations of every level-0 tile).  For each proxy
    cost = wB * border_iters + leaf_iters + kappa * (border_px + leaf_px)
the LPT deal (deal.lpt) is computed and every rank's tile list is timed on the GPU (host list,
CUDA events, L2 flushed); reported: max and mean rank time, max/mean and the speedup over the
1-GPU step.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402
from oracle import cache  # noqa: E402
from paper_2206_02255_b200 import deal  # noqa: E402


def timed(f, flush, reps):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        f()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="*", default=["C3", "C4", "C5"])
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for nm in a.workloads:
        w = W.CONFIGS[nm]
        rec = cache.tile_records(w.region, w.n, w.maxdwell, w.g, w.r, w.B, store=False)
        G = w.g * w.g
        bi = [sum(s["border_iters"] for s in rec["tiles"][t]["stats"]) for t in range(G)]
        li = [sum(s["leaf_iters"] for s in rec["tiles"][t]["stats"]) for t in range(G)]
        px = [sum(s["border_px"] + s["leaf_px"] for s in rec["tiles"][t]["stats"]) for t in range(G)]
        out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
        ws = mb.workspace(w.n, w.g, w.r, w.B)
        t1 = timed(lambda: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws), flush, a.reps)
        for wb in (1.0, 1.2, 1.5):
            for kappa in (0, 16, 64):
                cost = [wb * bi[t] + li[t] + kappa * px[t] for t in range(G)]
                parts = deal.lpt(cost, a.P)
                ts = [timed(lambda p=p: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=p),
                            flush, a.reps) for p in parts]
                print(json.dumps({"w": nm, "P": a.P, "wB": wb, "kappa": kappa, "t1_ms": round(t1, 4),
                                  "max_ms": round(max(ts), 4), "mean_ms": round(sum(ts) / len(ts), 4),
                                  "imbalance": round(max(ts) / (sum(ts) / len(ts)), 4),
                                  "speedup": round(t1 / max(ts), 3), "rank_ms": [round(x, 4) for x in ts]}),
                      flush=True)


if __name__ == "__main__":
    main()
