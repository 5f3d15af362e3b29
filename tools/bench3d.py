"""3-D ASK measurement (NEXT-4): tools/bench3d.py [V1 V2] [--reps 5]

Per configuration: device time (CUDA events, 256 MiB L2 flush between reps) of one
mandel3d_ask call and of the exhaustive 3-D kernel, Mvoxel/s, speedup, the fraction of voxels
where ASK differs from exhaustive, executed iterations (stats pass) and the FP32 rate of the
ASK call against the 148 x 128 x f_clk one-op-per-lane peak (6 FP32 instructions per iteration, R4').
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2206_02255_b200 import mandel3d as m3  # noqa: E402

PEAK = 148 * 128 * 1.965e9  # FP32 lane-ops/s at the max SM clock (bench.py's roofline basis)


def timed(fn, reps, flush):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts), sum(ts) / len(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["V1", "V2"])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in a.configs:
        w = W.CONFIGS3[name]
        vol = torch.empty((w.n, w.n, w.n), dtype=torch.int32, device="cuda")
        ex = torch.empty_like(vol)
        ws = m3.workspace3d(w.n, w.g, w.r, w.B)
        m3.ask3d(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=vol, ws=ws, stats=True)
        st = [s for s in m3.ask3d_stats(ws) if s["regions_in"]]
        iters = sum(s["border_iters"] + s["leaf_iters"] for s in st)
        t_ask, t_ask_mean = timed(lambda: m3.ask3d(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=vol, ws=ws),
                                  a.reps, flush)
        t_flat, _ = timed(lambda: m3.ask3d(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=ex, ws=ws, flat=True),
                          a.reps, flush)  # A/B: thread-per-voxel surface and leaf kernels
        same_flat = bool(torch.equal(ex, vol))
        t_ex, t_ex_mean = timed(lambda: m3.exhaustive3d(w.region, w.n, w.maxdwell, out=ex), max(2, a.reps // 2), flush)
        sum_ex = int(ex.sum(dtype=torch.int64).item())
        mism = int((vol != ex).sum().item())
        nv = w.n ** 3
        print(json.dumps({
            "config": w.as_dict(), "levels": len(st),
            "ask_ms": t_ask, "ask_ms_mean": t_ask_mean, "ex_ms": t_ex, "ex_ms_mean": t_ex_mean,
            "ask_flat_ms": t_flat, "flat_same_volume": same_flat,
            "ask_mvoxel_s": nv / t_ask / 1e3, "ex_mvoxel_s": nv / t_ex / 1e3, "speedup_vs_exhaustive": t_ex / t_ask,
            "mismatch_fraction_vs_exhaustive": mism / nv,
            "ask_executed_iters": iters, "ex_iters": sum_ex, "work_ratio": sum_ex / max(1, iters),
            "ask_fp32_frac": 6 * iters / (t_ask / 1e3) / PEAK, "ex_fp32_frac": 6 * sum_ex / (t_ex / 1e3) / PEAK,
            "level_stats": st}), flush=True)
        del vol, ex, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
