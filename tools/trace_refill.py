"""Timeline of the lane-refill kernels from a trace build (dev tool, GPU box):

    python tools/trace_refill.py [C3] [--P 8]      (builds /tmp/libmandel_trace.so itself)

For every traced launch (border levels, leaf) of the full image and of the heaviest rank of
a P-way deal: the active warps, the time from launch start to cursor exhaustion, and the
spread of warp end times after it (the level's tail), in microseconds.
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2206_02255_b200 import build  # noqa: E402

SO = "/tmp/libmandel_trace.so"
if os.environ.get("MANDEL_B200_LIB") != SO:
    extra = [d for d in os.environ.get("MANDEL_TRACE_DEFS", "").split(",") if d]
    build.build(out=SO, defines=["MANDEL_RF_TRACE"] + extra)
    os.environ["MANDEL_B200_LIB"] = SO
    os.execv(sys.executable, [sys.executable] + sys.argv)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_02255_b200 import _lib, deal  # noqa: E402


def fetch(lib):
    buf = np.zeros((16, 8192, 4), dtype=np.uint64)
    rc = lib.mandel_debug_rf_trace(buf.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0
    return buf


def summarize(buf, label):
    out = []
    live_all = buf[:, :, 2] > 0
    g0 = int(buf[:, :, 0][live_all].astype(np.int64).min()) if live_all.any() else 0
    for slot in range(16):
        t = buf[slot]
        live = t[:, 2] > 0
        if not live.any():
            continue
        t = t[live].astype(np.int64)
        t0 = t[:, 0].min()
        ex = t[:, 1][t[:, 1] > 0]
        ends = t[:, 2] - t0
        row = {"run": label, "kernel": "leaf" if slot == 15 else f"border{slot}",
               "active_warps": int(t[0, 3] >> 40), "px": int((t[:, 3] & ((1 << 40) - 1)).sum()),
               "first_exhaust_us": float((ex.min() - t0) / 1e3) if ex.size else None,
               "end_p50_us": float(np.percentile(ends, 50) / 1e3),
               "end_p90_us": float(np.percentile(ends, 90) / 1e3),
               "end_p99_us": float(np.percentile(ends, 99) / 1e3),
               "end_max_us": float(ends.max() / 1e3),
               "abs_start_us": float((t0 - g0) / 1e3), "abs_end_us": float((t[:, 2].max() - g0) / 1e3)}
        out.append(row)
        print(json.dumps(row), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="C3")
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--dtiles", action="store_true",
                    help="the heaviest rank of an LPT deal on exact costs through mandel_ask_dtiles with "
                         "sampled costs and overlapped fills (bench.py's N > 1 step); abs_* columns give gaps")
    a = ap.parse_args()
    lib = _lib.load()
    lib.mandel_debug_rf_trace.restype = ctypes.c_int
    lib.mandel_debug_rf_trace.argtypes = [ctypes.c_void_p]
    lib.mandel_debug_rf_trace_clear.restype = ctypes.c_int
    w = W.CONFIGS[a.workload]
    out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    costs = mb.preview_costs(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tile_cost=True)
    exact = mb.tile_costs(ws, w.g)
    heavy = max(deal.deal("costrank", w.g, a.P, costs), key=lambda p: sum(exact[k] for k in p))
    if a.dtiles:
        heavy = max(deal.deal("lpt", w.g, a.P, exact), key=lambda p: sum(exact[k] for k in p))
        dt = torch.tensor(heavy, dtype=torch.int32, device="cuda")
        dn = torch.tensor([len(heavy)], dtype=torch.int32, device="cuda")
        for label, kw in (("full", {}), (f"rank_of_{a.P}_dtiles", dict(dtiles=(dt, dn), tile_cost="sampled"))):
            for _ in range(2):
                mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, **kw)
            torch.cuda.synchronize()
            lib.mandel_debug_rf_trace_clear()
            mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, **kw)
            torch.cuda.synchronize()
            summarize(fetch(lib), label)
        return
    for label, tiles in (("full", None), (f"rank_of_{a.P}", heavy)):
        mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=tiles, serial=True)
        torch.cuda.synchronize()
        lib.mandel_debug_rf_trace_clear()
        mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=tiles, serial=True)
        torch.cuda.synchronize()
        summarize(fetch(lib), label)


if __name__ == "__main__":
    main()
