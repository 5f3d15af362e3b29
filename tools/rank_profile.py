"""Per-kernel efficiency of one rank's share vs the full image (single GPU, dev tool).

    python tools/rank_profile.py [C3] [--P 8] [--groups 1]

Runs the full image and the heaviest rank's tiles of a P-way cost-ranked deal, both with
serial fills and per-kernel events, and prints for every kernel: its time, its executed
iterations (stats pass), iterations per microsecond, and the rank/full ratio of that rate.
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


def run(w, out, ws, tiles, groups, reps=3):
    kw = dict(out=out, ws=ws, tiles=tiles, groups=groups, serial=True)
    mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, stats=True, **kw)
    st = mb.ask_stats(ws)
    for _ in range(2):
        mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, timing=True, **kw)
    torch.cuda.synchronize()
    acc = {}
    tot = 0.0
    for _ in range(reps):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, timing=True, **kw)
        e.record()
        e.synchronize()
        tot += s.elapsed_time(e) / reps
        for k in mb.kernel_times():
            key = (k["kind"], k["level"])
            acc[key] = acc.get(key, 0.0) + k["ms"] / reps
    work = {}
    for s_ in st:
        work[("b200_border", s_["level"])] = s_["border_iters"]
        if s_["leaf_iters"]:
            work[("b200_leaf", s_["level"])] = s_["leaf_iters"]
    return tot, acc, work, st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="C3")
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--groups", type=int, default=1)
    a = ap.parse_args()
    w = W.CONFIGS[a.workload]
    out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    costs = mb.preview_costs(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tile_cost=True)
    exact = mb.tile_costs(ws, w.g)
    parts = deal.deal("costrank", w.g, a.P, costs)
    heavy = max(parts, key=lambda p: sum(exact[k] for k in p))
    tf, kf, wf, stf = run(w, out, ws, None, a.groups)
    tr, kr, wr, str_ = run(w, out, ws, heavy, a.groups)
    print(json.dumps({"full_ms": tf, "rank_ms": tr, "ratio": tf / tr, "P": a.P,
                      "rank_work_frac": sum(exact[k] for k in heavy) / sum(exact)}))
    for key in kf:
        if key not in kr:
            continue
        row = {"kernel": f"{key[0]}:{key[1]}", "full_ms": round(kf[key], 4), "rank_ms": round(kr[key], 4)}
        if key in wf and wr.get(key):
            rf = wf[key] / (kf[key] * 1e3)
            rr = wr[key] / (kr[key] * 1e3)
            row.update({"full_it_per_us": round(rf / 1e6, 3), "rank_it_per_us": round(rr / 1e6, 3),
                        "work_frac": round(wr[key] / wf[key], 4), "rate_ratio": round(rr / rf, 3)})
        print(json.dumps(row))
    print(json.dumps({"full_levels": [s["regions_in"] for s in stf], "rank_levels": [s["regions_in"] for s in str_]}))


if __name__ == "__main__":
    main()
