"""Dev tool (GPU box): list pixels where mandel_ask differs from the oracle's ASK image.

    python tools/debug_mismatch.py [C1 ...] [--max 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
import paper_2206_02255_b200 as mb
import workloads as W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="*", default=["C1"])
    ap.add_argument("--max", type=int, default=20)
    a = ap.parse_args()
    print("lib", os.environ.get("MANDEL_B200_LIB", "in-tree"))
    for nm in a.workloads:
        w = W.CONFIGS[nm]
        out = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B).cpu().numpy()
        A, _ = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
        bad = np.argwhere(out != A)
        print(nm, "mismatches", len(bad), "sum gpu-orc", int((out.astype(np.int64) - A).sum()))
        for (i, j) in bad[: a.max]:
            print(f"  y={i} x={j} gpu={out[i, j]} oracle={A[i, j]} x%B={j % w.B} y%B={i % w.B}")


if __name__ == "__main__":
    main()
