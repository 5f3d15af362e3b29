"""Write the CPU oracle's per-tile digests of the BASELINE configurations to
tests/golden/oracle_tiles/ (TEST INFRASTRUCTURE; calls only oracle/).

    python tools/make_oracle_golden.py [C3 C4 C5 C2 C1 ...] [--procs N]

For each configuration every level-0 tile is run through the plain single-threaded oracle
(oracle.ask_tile), one process per core (oracle/cache.py); the SHA-256 of each tile's int32
image and its per-level statistics are stored under the key (region, n, maxdwell, g, r, B,
SHA-256 of oracle/*.c).  The GPU parity tests compare every pixel of the CUDA path's
full-size images with these digests.  index.json records, per configuration, the key, the
oracle's wall time, the core count and the summed CPU time.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import cache  # noqa: E402
import workloads as W  # noqa: E402


def configs(names):
    out = []
    for nm in names:
        if nm == "C2":
            out += W.c2_sweep()
        else:
            out.append(W.CONFIGS[nm])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["C1", "C2", "C3", "C5", "C4"])
    ap.add_argument("--procs", type=int, default=None)
    a = ap.parse_args()
    os.makedirs(cache.GOLDEN_DIR, exist_ok=True)
    idx_path = os.path.join(cache.GOLDEN_DIR, "index.json")
    index = json.load(open(idx_path)) if os.path.exists(idx_path) else {}
    for w in configs(a.names):
        key = cache.config_key(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
        path = os.path.join(cache.GOLDEN_DIR, key + ".json")
        if os.path.exists(path) and index.get(w.name, {}).get("key") == key:
            print(f"{w.name}: up to date ({key})", flush=True)
            continue
        t0 = time.perf_counter()
        tiles = cache.run_tiles(w.region, w.n, w.maxdwell, w.g, w.r, w.B, range(w.g * w.g), a.procs)
        wall = time.perf_counter() - t0
        procs = a.procs or len(os.sched_getaffinity(0))
        rec = {"config": {"region": [float(v) for v in w.region], "n": w.n, "maxdwell": w.maxdwell, "g": w.g,
                          "r": w.r, "B": w.B, "oracle_sha256": oracle.source_sha()},
               "tiles": tiles, "wall_s": round(wall, 3), "procs": procs}
        cache.save(rec, path)
        st = cache.summed_stats(rec)
        index[w.name] = {"key": key, "wall_s": round(wall, 3), "procs": procs,
                         "cpu_s": round(sum(t["cpu_s"] for t in tiles.values()), 3),
                         "executed_iters": sum(s["border_iters"] + s["leaf_iters"] for s in st),
                         "levels": len(st)}
        with open(idx_path, "w") as f:
            json.dump(index, f, indent=1, sort_keys=True)
        print(f"{w.name}: {len(tiles)} tiles, wall {wall:.1f} s on {procs} cores, "
              f"cpu {index[w.name]['cpu_s']:.1f} s", flush=True)


if __name__ == "__main__":
    main()
