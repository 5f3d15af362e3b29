"""Profiling driver (run under ncu on the GPU box): `warm` untimed ASK steps, then one more
ASK step, then one exhaustive launch, all on the bench.py launch configuration of a workload.

    python tools/prof_step.py [--workload C3] [--scheme b200] [--warm 1] [--no-ex]

One ASK step launches mandel_ask_kernel_count(...) kernels (one CUDA graph), so with ncu
`-s (warm * kernels_per_step) -c (kernels_per_step + 1)` captures exactly the last step and
the exhaustive kernel.  Prints the per-step kernel count to stderr.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2206_02255_b200 as mb
import workloads as W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--scheme", default="b200")
    ap.add_argument("--warm", type=int, default=1)
    ap.add_argument("--no-ex", action="store_true")
    ap.add_argument("--heavy-rank-of", type=int, default=0,
                    help="profile only the heaviest rank's tiles of a P-way cost-ranked deal")
    a = ap.parse_args()
    w = W.CONFIGS[a.workload]
    out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    kps = mb.kernel_count(w.n, w.g, w.r, w.B, a.scheme)
    print(f"kernels_per_step={kps}", file=sys.stderr)
    tiles = None
    if a.heavy_rank_of > 1:  # preview + exact-cost passes run before the profiled steps
        from paper_2206_02255_b200 import deal
        costs = mb.preview_costs(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
        mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, tile_cost=True)
        exact = mb.tile_costs(ws, w.g)
        parts = deal.deal("costrank", w.g, a.heavy_rank_of, costs)
        tiles = max(parts, key=lambda p: sum(exact[k] for k in p))
        torch.cuda.synchronize()
    for _ in range(a.warm + 1):
        mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws, scheme=a.scheme, tiles=tiles)
    torch.cuda.synchronize()
    if not a.no_ex:
        mb.exhaustive(w.region, w.n, w.maxdwell, out=out)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
