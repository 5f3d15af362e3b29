"""Quick device timing of Ex and ASK (both schemes) on the BASELINE workloads (dev tool)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2206_02255_b200 as mb
import workloads as W


def t_ms(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts), sum(ts) / len(ts)


def main():
    names = sys.argv[1:] or ["C1", "C3", "C5"]
    for nm in names:
        w = W.CONFIGS[nm]
        out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
        ws = mb.workspace(w.n, w.g, w.r, w.B)
        res = {"w": nm}
        res["ex_ms"] = t_ms(lambda: mb.exhaustive(w.region, w.n, w.maxdwell, out=out), reps=2, warm=1)
        for sch in ("b200", "sbr"):
            res[sch + "_ms"] = t_ms(lambda: mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, scheme=sch))
            mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, scheme=sch, stats=True)
            st = mb.ask_stats(ws)
            res[sch + "_iters"] = sum(s["border_iters"] + s["leaf_iters"] for s in st)
            res[sch + "_border_iters"] = sum(s["border_iters"] for s in st)
            res[sch + "_regions"] = [s["regions_in"] for s in st]
        res["speedup_b200"] = res["ex_ms"][0] / res["b200_ms"][0]
        res["speedup_sbr"] = res["ex_ms"][0] / res["sbr_ms"][0]
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
