"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck), run on the GPU box:

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py

Each scheme (b200, sbr, mbr; lane-refill and flat kernels; fills on a side stream and
serial; groups; tile subsets; stats / tile-cost passes), the exhaustive kernels, the Dynamic
Parallelism library and the 3-D library run on small inputs; every image is checked against
the CPU oracle, so the sanitizer sees exactly the paths the parity tests cover.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2206_02255_b200 as mb  # noqa: E402
import workloads as W  # noqa: E402
from paper_2206_02255_b200 import mandel3d as m3  # noqa: E402


def main():
    cases = [(W.SEAHORSE_REGION, 256, 700, 4, 2, 8), (W.NONDYADIC_REGIONS[0], 512, 1500, 8, 4, 4),
             (W.DEFAULT_REGION, 256, 300, 2, 2, 16),
             (W.SEAHORSE_REGION, 1024, 600, 2, 2, 32)]  # side-512 regions: block-per-region classify
    n_ok = 0
    for region, n, md, g, r, B in cases:
        A, _ = oracle.ask(region, n, md, g, r, B)
        E = oracle.exhaustive(region, n, md)
        for tuned in (False, True):
            assert np.array_equal(mb.exhaustive(region, n, md, tuned=tuned).cpu().numpy(), E)
            n_ok += 1
        ws = mb.workspace(n, g, r, B)
        variants = [dict(scheme=s) for s in ("b200", "sbr", "mbr")] + [
            dict(flat=True), dict(serial=True), dict(groups=3), dict(stats=True), dict(tile_cost=True),
            dict(tile_cost="sampled"), dict(timing=True), dict(timing="leaf")]
        for kw in variants:
            out = mb.ask(region, n, md, g, r, B, ws=ws, **kw)
            assert np.array_equal(out.cpu().numpy(), A), kw
            n_ok += 1
        tiles = list(range(0, g * g, 3))
        buf = torch.full((n, n), -1, dtype=torch.int32, device="cuda")
        mb.ask(region, n, md, g, r, B, out=buf, ws=ws, tiles=tiles)
        At, _ = oracle.ask(region, n, md, g, r, B, tiles=tiles)
        assert np.array_equal(buf.cpu().numpy(), At)
        n_ok += 1
        # device tile list chosen by the device deal (mandel_ask_dtiles + mandel_deal_lpt)
        costs = mb.tile_cost_view(ws, n, g, r, B).clone()
        dt = torch.full((g * g,), -1, dtype=torch.int32, device="cuda")
        dn = torch.zeros(1, dtype=torch.int32, device="cuda")
        mb.deal_lpt(costs, 3, 1, dt, dn)
        buf.fill_(-1)
        mb.ask(region, n, md, g, r, B, out=buf, ws=ws, dtiles=(dt, dn), tile_cost="sampled")
        torch.cuda.synchronize()
        mine = dt[: int(dn.item())].tolist()
        Ad, _ = oracle.ask(region, n, md, g, r, B, tiles=mine)
        assert np.array_equal(buf.cpu().numpy(), Ad)
        n_ok += 1
        # end to end into host memory: int32 and 16-bit images, whole (banded) and a tile subset
        h32 = torch.zeros(n * n, dtype=torch.int32).pin_memory()
        mb.ask_to_host(region, n, md, g, r, B, h32, buf, ws)
        assert np.array_equal(h32.numpy().reshape(n, n), A)
        h16 = torch.zeros(n * n, dtype=torch.uint16).pin_memory()
        mb.ask_to_host(region, n, md, g, r, B, h16, buf, ws)
        assert np.array_equal(h16.numpy().reshape(n, n).astype(np.int64), A)
        h16.zero_()
        mb.ask_to_host(region, n, md, g, r, B, h16, buf, ws, tiles=tiles)
        got = h16.numpy().reshape(n, n).astype(np.int64)
        assert np.array_equal(got[At != -1], At[At != -1])
        n_ok += 3
        if not os.environ.get("SANITIZE_NO_DP"):  # racecheck/synccheck/initcheck cannot follow CDP
            assert np.array_equal(mb.dp(region, n, md, g, r, B).cpu().numpy(), A)
            n_ok += 1
    A3, _ = oracle.ask3(W.DEFAULT_REGION3, 32, 128, 2, 2, 4)
    assert np.array_equal(m3.ask3d(W.DEFAULT_REGION3, 32, 128, 2, 2, 4).cpu().numpy(), A3)
    assert np.array_equal(m3.ask3d(W.DEFAULT_REGION3, 32, 128, 2, 2, 4, flat=True).cpu().numpy(), A3)
    torch.cuda.synchronize()
    mb.shutdown()
    print(f"sanitize driver: {n_ok + 2} invocations bit-exact vs the oracle")


if __name__ == "__main__":
    main()
