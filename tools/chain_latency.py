"""Latency of one dwell chain on B200 (dev tool, GPU box): the exhaustive kernel on a window
inside the main cardioid (every pixel runs maxdwell iterations) with few pixels, so each
chain's warp has its SM sub-partition (nearly) alone; time / maxdwell = cycles per iteration
of the dependent FMUL -> FADD -> FADD step.

    python tools/chain_latency.py [--maxdwell 2048]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--maxdwell", type=int, default=2048)
    a = ap.parse_args()
    clk = torch.cuda.clock_rate() if hasattr(torch.cuda, "clock_rate") else 1965
    for n in (16, 32, 64, 128, 256, 512):
        out = torch.empty((n, n), dtype=torch.int32, device="cuda")
        for _ in range(3):
            mb.exhaustive(W.INTERIOR_REGION, n, a.maxdwell, out=out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            mb.exhaustive(W.INTERIOR_REGION, n, a.maxdwell, out=out)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        t = min(ts)
        assert int(out.min()) == a.maxdwell
        warps = n * n // 32
        print(json.dumps({"n": n, "pixels": n * n, "warps": warps, "warps_per_smsp": warps / 592,
                          "ms": t, "cycles_per_iter_at_1965MHz": t * 1e-3 * 1.965e9 / a.maxdwell}), flush=True)


if __name__ == "__main__":
    main()
