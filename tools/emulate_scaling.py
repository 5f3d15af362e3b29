"""Single-GPU emulation of the P-rank strong-scaling step (the box has one B200).

    python tools/emulate_scaling.py C3 [--ranks 1,2,4,8] [--steps 4] [--reps 3]
                                       [--allreduce-us 20] [--plan feedback|preview]

Every rank of a P-way run executes the SAME work it would on its own GPU: its level-0 tiles
(mandel_ask_dtiles, tile list in device memory) on a full B200, so running the ranks one after
the other on one GPU and taking the slowest gives the P-GPU step time (the ranks share
nothing on the data path; the only cross-rank traffic is the g*g cost all-reduce below).

Plans (both device-resident):
  feedback  the steady-state frame loop of bench.py (DevicePlan.step): every SAMPLE_EVERY-th
            step renders with sampled per-tile cost counters (MANDEL_FLAG_TILE_COST_SAMPLED),
            the counters are all-reduced across ranks (here: summed over the ranks'
            workspaces; on the box: NCCL, modelled as --allreduce-us) and mandel_deal_lpt
            computes every rank's tiles on a side stream while the next step renders: the
            plan is overlapped, not added, as long as it is shorter than a step
            (plan_overlapped); the other steps render without counters.  The step time is the
            mean max-rank time over the last sampling period; the first steps are dealt on an
            n/32, maxdwell/8 preview.
  preview   every step is dealt on a fresh n/32, maxdwell/8 preview computed on every rank
            (ASK with tile costs + mandel_deal_lpt), its time charged.
Reported per P: max-over-ranks step time, the plan's charge, speedup over the 1-GPU step
(all tiles, no counters: bench.py's N=1 configuration), and a bit-exactness check of the
assembled image against that 1-GPU image.
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
from paper_2206_02255_b200 import multigpu  # noqa: E402


def ev_time(fn, flush):
    flush.zero_()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="C3")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=7)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--allreduce-us", type=float, default=20.0)
    ap.add_argument("--plan", default="feedback", choices=["feedback", "preview"])
    a = ap.parse_args()
    w = W.CONFIGS[a.workload]
    G = w.g * w.g
    out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ws1 = mb.workspace(w.n, w.g, w.r, w.B)
    one = lambda: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws1)  # noqa: E731
    one()
    t1 = statistics.median([ev_time(one, flush) for _ in range(a.reps)])
    ref = out.clone()
    res = {"workload": w.name, "plan": a.plan, "t1_ms": t1, "allreduce_us_model": a.allreduce_us, "P": {}}
    for P in [int(x) for x in a.ranks.split(",")]:
        ranks = [multigpu.DevicePlan(w, P, r, torch.device("cuda")) for r in range(P)]
        wss = [mb.workspace(w.n, w.g, w.r, w.B) for _ in range(P)]
        costs = torch.zeros(G, dtype=torch.int64, device="cuda")
        t_prev = ev_time(lambda: ranks[0].preview_costs(costs), flush)
        for rk in ranks:
            rk.deal(costs, both=True)
        steps = []
        for s in range(a.steps):
            out.fill_(-1)
            tr = []
            # feedback: as DevicePlan.step, only every SAMPLE_EVERY-th frame counts and re-deals
            sample = a.plan != "feedback" or s % multigpu.SAMPLE_EVERY == 0
            tc = ("sampled" if a.plan == "feedback" else True) if sample else False
            for rk, ws in zip(ranks, wss):
                f = lambda: rk.render(out, ws, tile_cost=tc)  # noqa: E731
                f()  # warm (graph capture on first use)
                tr.append(statistics.median([ev_time(f, flush) for _ in range(a.reps)]))
            if not sample:
                t_plan = 0.0
            elif a.plan == "feedback":  # all-reduce of the counters, then every rank's deal
                costs.zero_()
                for rk, ws in zip(ranks, wss):
                    costs += mb.tile_cost_view(ws, w.n, w.g, w.r, w.B)
                t_plan = statistics.median([ev_time(lambda: ranks[0].deal(costs), flush) for _ in range(a.reps)])
                t_plan += a.allreduce_us / 1e3 if P > 1 else 0.0
            else:
                t_plan = statistics.median([ev_time(lambda: ranks[0].preview_costs(costs), flush)
                                            for _ in range(a.reps)])
                t_plan += statistics.median([ev_time(lambda: ranks[0].deal(costs), flush) for _ in range(a.reps)])
            if sample:
                for rk in ranks:
                    rk.deal(costs, both=True)
            torch.cuda.synchronize()
            exact = bool(torch.equal(out, ref))
            steps.append({"rank_ms": tr, "max_rank_ms": max(tr), "plan_ms": t_plan, "bit_exact": exact,
                          "sampled": sample, "tiles": [int(rk.count.item()) for rk in ranks]})
        last = steps[-1]
        # feedback: the step time is the mean max-rank time over the last sampling period
        per = steps[-multigpu.SAMPLE_EVERY:] if a.plan == "feedback" else [last]
        max_rank = sum(x["max_rank_ms"] for x in per) / len(per)
        plan_ms = max(x["plan_ms"] for x in per)
        overlapped = a.plan == "feedback" and plan_ms < max_rank
        charged = max_rank + (plan_ms if P > 1 and not overlapped else 0.0)
        res["P"][P] = {"steps": steps, "charged_ms": charged, "speedup": t1 / charged, "plan_overlapped": overlapped,
                       "speedup_uncharged": t1 / max_rank,
                       "imbalance_time": last["max_rank_ms"] / (sum(last["rank_ms"]) / P),
                       "first_plan_preview_ms": t_prev}
        print(json.dumps({"P": P, "charged_ms": round(charged, 4), "speedup": round(t1 / charged, 3),
                          "max_rank_ms": round(max_rank, 4), "plan_ms": round(plan_ms, 4),
                          "plan_overlapped": overlapped,
                          "imbalance_time": round(res["P"][P]["imbalance_time"], 4),
                          "bit_exact": last["bit_exact"],
                          "step_max_rank_ms": [round(x["max_rank_ms"], 4) for x in steps]}), flush=True)
        del wss
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
