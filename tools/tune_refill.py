"""Sweep the lane-refill knobs on the GPU box: one library variant per point, built into /tmp
with extra -D defines, timed with tools/ab.py (MANDEL_B200_LIB points the binding at it).

    python tools/tune_refill.py [C3 C5] [--points "RFL_K=32,RFL_T=4;RFL_K=16,RFL_T=8"]

Knobs (ask_kernels.cuh): MANDEL_RFB_{K,T,CH} (border kernels), MANDEL_RFL_{K,T,CH} (leaf),
MANDEL_RF_MINB (resident blocks per SM).  An empty point is the in-tree default.
"""
import argparse
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2206_02255_b200 import build  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="*", default=["C3"])
    ap.add_argument("--points", default="")
    ap.add_argument("--variants", default="b200")
    a = ap.parse_args()
    for pt in a.points.split(";"):
        defs = [f"MANDEL_{d.strip()}" for d in pt.split(",") if d.strip()]
        tag = hashlib.md5(pt.encode()).hexdigest()[:8]
        so = f"/tmp/libmandel_{tag}.so"
        build.build(out=so, defines=defs)
        env = dict(os.environ, MANDEL_B200_LIB=so)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ab.py"), *a.workloads,
                            "--variants", a.variants, "--reps", "3"], env=env, capture_output=True, text=True)
        print(f"[{pt or 'default'}]", r.stdout.strip(), r.stderr.strip()[-300:], flush=True)


if __name__ == "__main__":
    main()
