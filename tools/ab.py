"""A/B device timing of ASK variants on BASELINE workloads (dev tool, GPU box).

    python tools/ab.py [C3 C5 ...] [--reps 5] [--variants b200,flat,sbr]

Per variant: mean/min step ms over `reps` graph launches (L2 flushed between), per-kernel
ms (graph event nodes), executed iterations, and a bit-exact check against the first
variant's image.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2206_02255_b200 as mb
import workloads as W

VARIANTS = {"b200": dict(scheme="b200"), "flat": dict(scheme="b200", flat=True), "sbr": dict(scheme="sbr"), "mbr": dict(scheme="mbr"),
            "serial": dict(scheme="b200", serial=True), "mbr_serial": dict(scheme="mbr", serial=True),
            "g2": dict(scheme="b200", groups=2), "g4": dict(scheme="b200", groups=4),
            "g8": dict(scheme="b200", groups=8), "g1": dict(scheme="b200", groups=1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="*", default=["C3", "C5"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", default="b200,serial,flat,sbr")
    ap.add_argument("--ex", action="store_true")
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for nm in a.workloads:
        w = W.CONFIGS[nm]
        out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
        ref = None
        ws = mb.workspace(w.n, w.g, w.r, w.B)
        res = {"w": nm, "lib": os.environ.get("MANDEL_B200_LIB", "in-tree")}
        if a.ex:
            mb.exhaustive(w.region, w.n, w.maxdwell, out=out)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record(); mb.exhaustive(w.region, w.n, w.maxdwell, out=out); e.record(); e.synchronize()
            res["ex_ms"] = s.elapsed_time(e)
        for v in a.variants.split(","):
            if v == "dp":  # Dynamic Parallelism baseline (libmandel_dp.so): device time only
                mb.dp(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out)
                torch.cuda.synchronize()
                same = True if ref is None else bool(torch.equal(ref, out))
                ts = []
                for _ in range(a.reps):
                    flush.zero_()
                    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                    s.record()
                    mb.dp(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out)
                    e.record(); e.synchronize()
                    ts.append(s.elapsed_time(e))
                res[v] = {"ms_mean": sum(ts) / len(ts), "ms_min": min(ts), "same_image": same}
                continue
            kw = VARIANTS[v]
            mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, stats=True, **kw)
            st = mb.ask_stats(ws)
            iters = sum(x["border_iters"] + x["leaf_iters"] for x in st)
            img = out.clone() if ref is None else out
            if ref is None:
                ref = img
                same = True
            else:
                same = bool(torch.equal(ref, out))
            for _ in range(2):
                mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, timing=True, **kw)
            ts, kt = [], {}
            for _ in range(a.reps):
                flush.zero_()
                s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                s.record()
                mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, timing=True, **kw)
                e.record(); e.synchronize()
                ts.append(s.elapsed_time(e))
                for k in mb.kernel_times():
                    kt[k["kind"]] = kt.get(k["kind"], 0.0) + k["ms"] / a.reps
            tn = []
            mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, **kw)  # capture this graph
            torch.cuda.synchronize()
            for _ in range(a.reps):
                flush.zero_()
                s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                s.record()
                mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, **kw)
                e.record(); e.synchronize()
                tn.append(s.elapsed_time(e))
            res[v] = {"ms_mean": sum(ts) / len(ts), "ms_min": min(ts), "iters": iters,
                      "ms_notiming_mean": sum(tn) / len(tn),
                      "giter_s_exec": iters / (min(ts) / 1e3) / 1e9, "same_image": same,
                      "kernels": {k: round(x, 4) for k, x in kt.items()}}
        print(json.dumps(res), flush=True)
        del out, ref, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
