"""Launch-list driver (run under ncu): one 8-way-rank ASK step of C3 with the rank's tiles as a
host list, then the same step with the device list (mandel_ask_dtiles), each after one warm
call.  Compare the two launch lists kernel by kernel (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_02255_b200 import multigpu  # noqa: E402

w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
ws = mb.workspace(w.n, w.g, w.r, w.B)
plan = multigpu.DevicePlan(w, 8, 0, torch.device("cuda"))
mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tile_cost=True)
plan.deal(mb.tile_cost_view(ws, w.n, w.g, w.r, w.B).clone(), both=True)
host = plan.host_tiles()
torch.cuda.synchronize()
for _ in range(2):
    mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tiles=host)
torch.cuda.synchronize()
for _ in range(2):
    mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, dtiles=(plan.tiles, plan.count))
torch.cuda.synchronize()
print("kernels per step", mb.kernel_count(w.n, w.g, w.r, w.B), file=sys.stderr)
