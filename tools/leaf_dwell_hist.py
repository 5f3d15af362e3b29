"""Dwell distribution of the pixels the B200 scheme computes (leaf interiors and new ring
pixels), from the GPU exhaustive image and a vectorised replay of the ASK decisions in torch
(dev tool, GPU box).  Used to size a short-pixel prepass.

    python tools/leaf_dwell_hist.py [C3]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2206_02255_b200 as mb
import workloads as W


def ring_minmax(E, d):
    n = E.shape[0]
    k = n // d
    top = E[0::d, :].reshape(k, k, d)
    bot = E[d - 1::d, :].reshape(k, k, d)
    left = E[:, 0::d].reshape(k, d, k).transpose(1, 2)
    right = E[:, d - 1::d].reshape(k, d, k).transpose(1, 2)
    lo = torch.minimum(torch.minimum(top.amin(2), bot.amin(2)), torch.minimum(left.amin(2), right.amin(2)))
    hi = torch.maximum(torch.maximum(top.amax(2), bot.amax(2)), torch.maximum(left.amax(2), right.amax(2)))
    return lo, hi


def main():
    nm = sys.argv[1] if len(sys.argv) > 1 else "C3"
    w = W.CONFIGS[nm]
    n = w.n
    # the ASK image: ring decisions are made on ASK's own ring values, which equal Ex's
    A = mb.ask(w.region, n, w.maxdwell, w.g, w.r, w.B)
    d = n // w.g
    active = torch.ones((w.g, w.g), dtype=torch.bool, device="cuda")
    edges = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]
    leaf_hist = torch.zeros(len(edges) + 1, dtype=torch.int64, device="cuda")
    while True:
        lo, hi = ring_minmax(A, d)
        uni = lo == hi
        sub = active & ~uni
        if d // w.r >= w.B:
            active = sub.repeat_interleave(w.r, 0).repeat_interleave(w.r, 1)
            d //= w.r
            continue
        # leaves: interiors of non-uniform regions at this level
        k = n // d
        blocks = A.reshape(k, d, k, d).permute(0, 2, 1, 3)[:, :, 1:d - 1, 1:d - 1]
        vals = blocks[sub]  # (leaves, d-2, d-2)
        v = vals.reshape(-1)
        b = torch.bucketize(v, torch.tensor(edges, device="cuda"), right=True)
        leaf_hist += torch.bincount(b, minlength=len(edges) + 1)
        break
    tot = int(leaf_hist.sum())
    cum = torch.cumsum(leaf_hist, 0).tolist()
    out = {"w": nm, "leaf_px": tot, "le": {f"<={e}": cum[i + 1] / tot for i, e in enumerate(edges) if i + 1 < len(cum)},
           "mean": float(v.double().mean()), "median": float(v.double().median())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
