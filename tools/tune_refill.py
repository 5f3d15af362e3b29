"""Sweep the lane-refill knobs (MANDEL_RF_K, MANDEL_RF_T, MANDEL_RF_CH) on the GPU box:
builds one library variant per point into /tmp and times tools/ab.py with it.

    python tools/tune_refill.py [C3] [--points K:T:CH,...]
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2206_02255_b200 import build  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="*", default=["C3"])
    ap.add_argument("--points", default="8:8:128,8:4:128,8:16:128,8:1:128,4:8:128,16:8:128,8:8:32,8:8:512")
    a = ap.parse_args()
    for pt in a.points.split(","):
        K, T, CH = pt.split(":")
        so = f"/tmp/libmandel_K{K}_T{T}_CH{CH}.so"
        build.build(out=so, defines=[f"MANDEL_RF_K={K}", f"MANDEL_RF_T={T}", f"MANDEL_RF_CH={CH}"])
        env = dict(os.environ, MANDEL_B200_LIB=so)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ab.py"), *a.workloads,
                            "--variants", "b200", "--reps", "3"], env=env, capture_output=True, text=True)
        print(f"K={K} T={T} CH={CH}", r.stdout.strip(), r.stderr.strip()[-300:], flush=True)


if __name__ == "__main__":
    main()
