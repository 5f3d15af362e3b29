"""Where the multi-GPU deal's preview time goes (dev tool, GPU box): device time of the preview
ASK call with and without per-tile cost counters, and the host wall time of preview_costs()."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402

for name in ("C3", "C5", "C4"):
    w = W.CONFIGS[name]
    for sh, dsh in ((8, 2), (16, 8)):
        pn, pB, pmd = w.n // sh, max(2, w.B // sh), max(1, w.maxdwell // dsh)
        ws = mb.workspace(pn, w.g, w.r, pB)
        out = torch.empty((pn, pn), dtype=torch.int32, device="cuda")
        res = {"w": name, "preview": [sh, dsh]}
        for tc in (False, True):
            f = lambda: mb.ask(w.region, pn, pmd, w.g, w.r, pB, out=out, ws=ws, tile_cost=tc)  # noqa: E731
            f()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            f()
            e.record()
            e.synchronize()
            res["ask_ms_tile_cost" if tc else "ask_ms_plain"] = s.elapsed_time(e)
        mb.preview_costs(w.region, w.n, w.maxdwell, w.g, w.r, w.B, shrink=sh, dwell_shrink=dsh)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mb.preview_costs(w.region, w.n, w.maxdwell, w.g, w.r, w.B, shrink=sh, dwell_shrink=dsh)
        res["preview_costs_wall_ms"] = 1e3 * (time.perf_counter() - t0)
        print(json.dumps(res), flush=True)
