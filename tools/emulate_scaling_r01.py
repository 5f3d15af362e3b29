"""Single-GPU emulation of the multi-GPU strong-scaling run (BASELINE config 3: n=32768 on
1/2/4/8 B200, north_star target >= 7x from 1 to 8).

Level-0 tiles are independent and the hot path has no collective, so a rank's
step is exactly mandel_ask_tiles over its dealt tiles; this tool runs every rank's tile set on
the one GPU of the box, one after another, and reports the max over ranks of the per-rank
device time (what bench.py measures under torchrun) plus the imbalance of each deal.

    python tools/emulate_scaling.py [C3] [--ranks 1,2,4,8] [--deals costrank,cyclic,diagonal]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_02255_b200 import deal  # noqa: E402


GROUPS = None
SCHEME = "b200"


def time_tiles(w, out, ws, tiles, flush, reps):
    f = lambda: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=tiles,  # noqa: E731
                       groups=GROUPS, scheme=SCHEME)
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
    return sum(ts) / len(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="C3")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--deals", default="lpt,costrank,cyclic,diagonal")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--groups", type=int, default=None)
    ap.add_argument("--scheme", default="b200")
    ap.add_argument("--preview", default="8,2", help="preview shrink,dwell_shrink")
    a = ap.parse_args()
    global GROUPS, SCHEME
    GROUPS = a.groups
    SCHEME = a.scheme
    w = W.CONFIGS[a.workload]
    out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sh, dsh = (int(x) for x in a.preview.split(","))
    costs = mb.preview_costs(w.region, w.n, w.maxdwell, w.g, w.r, w.B, shrink=sh, dwell_shrink=dsh)
    torch.cuda.synchronize()
    t0 = time.perf_counter()  # warm (the first call captured the preview graph)
    costs = mb.preview_costs(w.region, w.n, w.maxdwell, w.g, w.r, w.B, shrink=sh, dwell_shrink=dsh)
    torch.cuda.synchronize()
    preview_ms = 1e3 * (time.perf_counter() - t0)
    # exact per-tile costs (executed iterations) from one full-size counter pass
    mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tile_cost=True)
    exact = mb.tile_costs(ws, w.g)
    t1 = time_tiles(w, out, ws, None, flush, a.reps)
    res = {"workload": w.name, "preview": a.preview, "scheme": SCHEME, "groups": GROUPS, "t1_ms": t1, "preview_ms": preview_ms, "deals": {}}
    for dname in a.deals.split(","):
        for P in [int(x) for x in a.ranks.split(",")]:
            # "<deal>_exact": dealt on the exact per-tile costs (the estimator's upper bound)
            base = dname[:-6] if dname.endswith("_exact") else dname
            est = exact if dname.endswith("_exact") else costs
            parts = deal.deal(base, w.g, P, est if base in ("costrank", "lpt") else None)
            per = [time_tiles(w, out, ws, p, flush, a.reps) for p in parts]
            tmax = max(per)
            res["deals"][f"{dname}:{P}"] = {
                "max_rank_ms": tmax, "mean_rank_ms": sum(per) / P, "speedup_vs_1": t1 / tmax,
                "imbalance_time": tmax / (sum(per) / P), "imbalance_exact_iters": deal.imbalance(parts, exact)}
            print(json.dumps({"deal": dname, "P": P, **res["deals"][f"{dname}:{P}"]}), flush=True)
    # per-kernel breakdown of the heaviest rank at the largest P (costrank deal)
    P = max(int(x) for x in a.ranks.split(","))
    parts = deal.deal("costrank", w.g, P, costs)
    heavy = max(parts, key=lambda p: sum(exact[k] for k in p))
    for _ in range(2):
        mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=heavy, timing=True, groups=GROUPS,
               scheme=SCHEME)
    torch.cuda.synchronize()
    res["heavy_rank_kernels"] = [dict(k) for k in mb.kernel_times()]
    mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, timing=True, scheme=SCHEME)
    torch.cuda.synchronize()
    res["full_kernels"] = [dict(k) for k in mb.kernel_times()]
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
