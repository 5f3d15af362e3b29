"""Block-shape sweep of the exhaustive kernel (the paper tunes Ex's block per GPU):
one library build per shape (-DMANDEL_EX_BX/BY), timed on the given workloads.

    python tools/tune_ex.py [C3 C5] [--shapes 16x16,32x8,...]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2206_02255_b200 import build  # noqa: E402

CHILD = r"""
import json, sys, torch
sys.path.insert(0, %r)
import paper_2206_02255_b200 as mb, workloads as W
res = {}
for nm in %r:
    w = W.CONFIGS[nm]
    out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
    mb.exhaustive(w.region, w.n, w.maxdwell, out=out); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); mb.exhaustive(w.region, w.n, w.maxdwell, out=out); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    res[nm] = min(ts)
    del out
print(json.dumps(res))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="*", default=["C3", "C5"])
    ap.add_argument("--shapes", default="16x16,32x8,8x32,32x4,64x4,32x16,16x8,128x2,32x2")
    a = ap.parse_args()
    for sh in a.shapes.split(","):
        bx, by = sh.split("x")
        so = f"/tmp/libmandel_ex_{bx}x{by}.so"
        build.build(out=so, defines=[f"MANDEL_EX_BX={bx}", f"MANDEL_EX_BY={by}"])
        env = dict(os.environ, MANDEL_B200_LIB=so)
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, a.workloads)], env=env, capture_output=True,
                           text=True)
        print(json.dumps({"shape": sh, "ms": json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0
                          else r.stderr[-300:]}), flush=True)


if __name__ == "__main__":
    main()
