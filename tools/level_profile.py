"""Per-level efficiency of the B200 scheme (dev tool, GPU box): for each level, the new border
pixels, their iterations, the border kernel's device time (graph event nodes) and the
resulting iteration rate, next to the leaf kernel's; shows where level tails cost time.

    python tools/level_profile.py [C3 ...] [--reps 5] [--tiles-of P]   (P: heaviest rank of a P-way deal)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2206_02255_b200 as mb
import workloads as W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="*", default=["C3"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tiles-of", type=int, default=0)
    a = ap.parse_args()
    for nm in a.workloads:
        w = W.CONFIGS[nm]
        out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
        ws = mb.workspace(w.n, w.g, w.r, w.B)
        tiles = None
        if a.tiles_of > 1:
            from paper_2206_02255_b200 import deal
            costs = mb.preview_costs(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
            parts = deal.deal("costrank", w.g, a.tiles_of, costs)
            tiles = max(parts, key=lambda p: sum(costs[k] for k in p))
        mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=tiles, stats=True)
        st = [s for s in mb.ask_stats(ws) if s["regions_in"] > 0]
        acc = {}
        for _ in range(a.reps):
            mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=tiles, timing=True)
            torch.cuda.synchronize()
            for k in mb.kernel_times():
                key = (k["kind"], k["level"])
                acc[key] = acc.get(key, 0.0) + k["ms"] / a.reps
        rows = []
        leaf_rate = None
        for s in st:
            l = s["level"]
            t = acc.get(("b200_border", l), 0.0)
            tc = acc.get(("b200_classify", l), 0.0)
            rows.append({"level": l, "side": s["side"], "regions": s["regions_in"], "border_px": s["border_px"],
                         "border_iters": s["border_iters"], "border_ms": round(t, 4), "classify_ms": round(tc, 4),
                         "giter_s": round(s["border_iters"] / (t / 1e3) / 1e9, 1) if t else None,
                         "fill_ms": round(acc.get(("fill", l), 0.0), 4)})
        lt = acc.get(("b200_leaf", st[-1]["level"]), 0.0)
        li = sum(s["leaf_iters"] for s in st)
        leaf_rate = li / (lt / 1e3) / 1e9 if lt else None
        res = {"w": nm, "tiles": len(tiles) if tiles else w.g * w.g, "levels": rows, "leaf_ms": round(lt, 4),
               "leaf_iters": li, "leaf_giter_s": round(leaf_rate, 1) if leaf_rate else None}
        # time the border levels would take at the leaf kernel's rate
        res["border_ms_total"] = round(sum(r["border_ms"] for r in rows), 4)
        res["border_ms_at_leaf_rate"] = round(sum(r["border_iters"] for r in rows) / (leaf_rate * 1e9) * 1e3, 4) \
            if leaf_rate else None
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
