"""One rank's share through the call paths the multi-GPU step can use (dev tool, GPU box):
the heaviest rank of a P-way LPT deal on exact tile costs, timed (CUDA events, L2 flushed,
median of reps) as
  host        mandel_ask_tiles with a host tile list, no counters (tools/ab_variants.py C3r8)
  host+s      the same with the sampled per-tile cost counters (MANDEL_FLAG_TILE_COST_SAMPLED)
  dtiles      mandel_ask_dtiles (tile list and count in device memory), no counters
  dtiles+s    mandel_ask_dtiles with the sampled counters (bench.py's N > 1 step)
plus the 1-GPU step, so the difference between the paths shows what the device-resident plan
costs a rank.

    python tools/rank_paths.py [C3 C4 ...] [--P 8] [--reps 7]
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
    ap.add_argument("workloads", nargs="*", default=["C3"])
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for nm in a.workloads:
        w = W.CONFIGS[nm]
        out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
        ws = mb.workspace(w.n, w.g, w.r, w.B)
        ask = lambda **kw: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, **kw)  # noqa: E731
        t1 = timed(lambda: ask(), flush, a.reps)
        ask(tile_cost=True)
        exact = mb.tile_costs(ws, w.g)
        parts = deal.deal("lpt", w.g, a.P, exact)
        tiles = max(parts, key=lambda p: sum(exact[k] for k in p))
        dt = torch.tensor(tiles, dtype=torch.int32, device="cuda")
        dn = torch.tensor([len(tiles)], dtype=torch.int32, device="cuda")
        res = {"w": nm, "P": a.P, "t1_ms": t1, "rank_tiles": len(tiles)}
        res["host"] = timed(lambda: ask(tiles=tiles), flush, a.reps)
        res["host+s"] = timed(lambda: ask(tiles=tiles, tile_cost="sampled"), flush, a.reps)
        res["dtiles"] = timed(lambda: ask(dtiles=(dt, dn)), flush, a.reps)
        res["dtiles+s"] = timed(lambda: ask(dtiles=(dt, dn), tile_cost="sampled"), flush, a.reps)
        for k in ("host", "host+s", "dtiles", "dtiles+s"):
            res[k] = round(res[k], 4)
            res["speedup_" + k] = round(t1 / res[k], 3)
        def kern(**kw):
            ask(timing=True, **kw)
            torch.cuda.synchronize()
            kd = {}
            for k in mb.kernel_times():
                key = k["kind"] if k["kind"] in ("init", "fill") else f"{k['kind'][5:]}{k['level']}"
                kd[key] = round(kd.get(key, 0.0) + k["ms"], 4)
            return kd
        res["kernels_host"] = kern(tiles=tiles)
        res["kernels_host+s"] = kern(tiles=tiles, tile_cost="sampled")
        res["kernels_dtiles"] = kern(dtiles=(dt, dn))
        res["kernels_dtiles+s"] = kern(dtiles=(dt, dn), tile_cost="sampled")
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
