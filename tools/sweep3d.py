"""3-D {g, r, B} sweep (NEXT-4; the k = 3 analogue of BASELINE config 2): device time of
mandel3d_ask over g in {2,4,8,16} x r in {2,4} x B in {4,8,16,32} at n = 512, maxdwell 512,
beside the 3-D exhaustive kernel; executed iterations from the counter pass.

    python tools/sweep3d.py [--n 512] [--maxdwell 512]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2206_02255_b200 import mandel3d as m3  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--maxdwell", type=int, default=512)
    a = ap.parse_args()
    n, md, reg = a.n, a.maxdwell, W.DEFAULT_REGION3
    vol = torch.empty((n, n, n), dtype=torch.int32, device="cuda")
    t_ex = timed(lambda: m3.exhaustive3d(reg, n, md, out=vol))
    rows = []
    for g in (2, 4, 8, 16):
        for r in (2, 4):
            for B in (4, 8, 16, 32):
                if g * B > n or m3.levels3d(n, g, r, B) == 0:
                    continue
                ws = m3.workspace3d(n, g, r, B)
                m3.ask3d(reg, n, md, g, r, B, out=vol, ws=ws, stats=True)
                st = [s for s in m3.ask3d_stats(ws) if s["regions_in"]]
                it = sum(s["border_iters"] + s["leaf_iters"] for s in st)
                t = timed(lambda: m3.ask3d(reg, n, md, g, r, B, out=vol, ws=ws))
                row = {"g": g, "r": r, "B": B, "levels": len(st), "leaf_side": st[-1]["side"], "ms": t,
                       "speedup_vs_ex": t_ex / t, "executed_iters": it}
                rows.append(row)
                print(json.dumps(row), flush=True)
                del ws
    best = min(rows, key=lambda x: x["ms"])
    print(json.dumps({"n": n, "maxdwell": md, "ex_ms": t_ex, "best": best}), flush=True)


if __name__ == "__main__":
    main()
