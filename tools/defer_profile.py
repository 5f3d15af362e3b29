"""Per-level profile of the deferred-pixel mode (MANDEL_FLAG_DEFER) on one
rank's share of a cost-ranked 8-way deal and on the full image (dev tool, GPU box).

    python tools/defer_profile.py [C3] [--caps 0,256] [--P 8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_02255_b200 import deal  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="C3")
    ap.add_argument("--caps", default="0,256")
    ap.add_argument("--P", type=int, default=8)
    a = ap.parse_args()
    w = W.CONFIGS[a.workload]
    out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    costs = mb.preview_costs(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    parts = deal.deal("costrank", w.g, a.P, costs)
    heavy = max(parts, key=lambda p: sum(costs[k] for k in p))
    for share, tiles in (("rank", heavy), ("full", None)):
        for cap in [int(c) for c in a.caps.split(",")]:
            kw = dict(out=out, ws=ws, tiles=tiles, defer=cap)
            for _ in range(3):
                mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, timing=True, **kw)
            torch.cuda.synchronize()
            kts = mb.kernel_times()
            mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, **kw)
            st = mb.ask_stats(ws)
            lv = []
            for s in st:
                if s["regions_in"] == 0:
                    continue
                l = s["level"]
                lv.append({"level": l, "side": s["side"], "regions": s["regions_in"], "deferred": s["deferred"],
                           "uncertain": s["uncertain"], "unc_px": s["uncertain"] * (4 * s["side"] - 4),
                           "ms": {k["kind"]: round(sum(x["ms"] for x in kts if x["kind"] == k["kind"] and x["level"] == l), 4)
                                  for k in kts if k["level"] == l}})
            tot = {}
            for k in kts:
                tot[k["kind"]] = round(tot.get(k["kind"], 0.0) + k["ms"], 4)
            print(json.dumps({"w": w.name, "share": share, "cap": cap, "totals": tot, "levels": lv}), flush=True)


if __name__ == "__main__":
    main()
