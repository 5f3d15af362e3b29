"""Two 3-D ASK calls (warm-up + profiled) for ncu launch lists (dev tool, GPU box):
    ncu --metrics gpu__time_duration.sum -s 14 -c 14 python tools/prof3d.py V2 [--flat]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2206_02255_b200 import mandel3d as m3  # noqa: E402

w = W.CONFIGS3[sys.argv[1] if len(sys.argv) > 1 else "V2"]
flat = "--flat" in sys.argv
vol = torch.empty((w.n, w.n, w.n), dtype=torch.int32, device="cuda")
ws = m3.workspace3d(w.n, w.g, w.r, w.B)
for _ in range(2):
    m3.ask3d(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=vol, ws=ws, flat=flat)
torch.cuda.synchronize()
