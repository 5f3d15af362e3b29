"""Exact dwell census of the pixels the B200 scheme computes (dev tool, GPU box): per level
the new ring pixels (the union of the level's rings minus every earlier level's), and the leaf
interiors, as bincounts over dwell 1..maxdwell.  Drives the chunk/replay cost model of the
refill engines (tools/engine_model.py).

    python tools/dwell_census.py C3 [C5 ...] > profiles/r02_dwell_census.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from leaf_dwell_hist import ring_minmax  # noqa: E402


def census(nm):
    w = W.CONFIGS[nm]
    n, md = w.n, w.maxdwell
    A = mb.ask(w.region, n, md, w.g, w.r, w.B)
    torch.cuda.synchronize()
    dev = A.device
    seen = torch.zeros((n, n), dtype=torch.bool, device=dev)
    ar = torch.arange(n, device=dev)
    d = n // w.g
    active = torch.ones((w.g, w.g), dtype=torch.bool, device=dev)
    level = 0
    out = {"w": nm, "n": n, "maxdwell": md, "border": [], "leaf": None}
    while True:
        k = n // d
        line = (ar % d == 0) | (ar % d == d - 1)
        act = active.repeat_interleave(d, 0).repeat_interleave(d, 1)
        ring = (line[:, None] | line[None, :]) & act
        new = ring & ~seen
        seen |= ring
        del ring
        v = A[new]
        bc = torch.bincount(v, minlength=md + 1).tolist()
        out["border"].append({"level": level, "d": d, "regions": int(active.sum()), "px": int(v.numel()),
                              "hist": {i: c for i, c in enumerate(bc) if c}})
        del new, act, v
        lo, hi = ring_minmax(A, d)
        sub = active & (lo != hi)
        if d // w.r >= w.B:
            active = sub.repeat_interleave(w.r, 0).repeat_interleave(w.r, 1)
            d //= w.r
            level += 1
            continue
        blocks = A.reshape(k, d, k, d).permute(0, 2, 1, 3)[:, :, 1:d - 1, 1:d - 1]
        v = blocks[sub].reshape(-1)
        bc = torch.bincount(v, minlength=md + 1).tolist()
        out["leaf"] = {"level": level, "d": d, "leaves": int(sub.sum()), "px": int(v.numel()),
                       "hist": {i: c for i, c in enumerate(bc) if c}}
        break
    return out


def main():
    for nm in sys.argv[1:] or ["C3"]:
        print(json.dumps(census(nm)), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
