"""Tile-parallel runner and on-disk cache of the CPU oracle's ASK images — TEST
INFRASTRUCTURE ONLY (tests/, tools/make_oracle_golden.py; never the product path).

The oracle itself stays the plain single-threaded C recursion of mandel_oracle.c.  What this
module adds is bookkeeping around it, none of the method's arithmetic:

  * parallelism: level-0 regions never interact (every ASK decision is local to a region,
    P:366-377), so the image of a configuration is the union of independent per-tile oracle
    runs (oracle.ask_tile, one level-0 tile each -- pinned equal to the matching slice of the
    whole-image oracle.ask by tests/test_oracle_pins.py); one single-threaded process per host
    core runs them;
  * a digest per tile: SHA-256 of the tile's (d0, d0) int32 image in C order (little-endian),
    plus the tile's per-level statistics, so that a full-size image (4 GiB at C3, 16 GiB at
    C4) can be compared bit for bit without keeping the oracle's image;
  * a cache keyed by (region, n, maxdwell, g, r, B, oracle.source_sha()): first the committed
    golden files under tests/golden/oracle_tiles/ (written by tools/make_oracle_golden.py,
    which calls only oracle/), then $ORACLE_CACHE_DIR (default <repo>/.oracle_cache, not
    tracked), else computed here and stored in the latter.  A change to the oracle's C source
    changes the key, so stale results are never used.
"""
from __future__ import annotations

import hashlib
import json
import os
import time
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import ask_tile, build, source_sha

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden", "oracle_tiles")
STAT_KEYS = ("regions_in", "filled", "subdivided", "leaves", "border_px", "border_iters", "leaf_px", "leaf_iters")


def cache_dir() -> str:
    return os.environ.get("ORACLE_CACHE_DIR") or os.path.join(ROOT, ".oracle_cache")


def tile_digest(img: np.ndarray) -> str:
    """SHA-256 of a tile image as little-endian int32 in C order."""
    a = np.ascontiguousarray(img, dtype="<i4")
    return hashlib.sha256(a.tobytes()).hexdigest()


def config_key(region, n: int, maxdwell: int, g: int, r: int, B: int, oracle_sha: Optional[str] = None) -> str:
    desc = json.dumps({"region": [float(v).hex() for v in region], "n": int(n), "maxdwell": int(maxdwell),
                       "g": int(g), "r": int(r), "B": int(B), "oracle": oracle_sha or source_sha()},
                      sort_keys=True)
    return hashlib.sha256(desc.encode()).hexdigest()[:32]


def _one_tile(args):
    region, n, md, g, r, B, t = args
    t0 = time.perf_counter()
    img, st = ask_tile(region, n, md, g, r, B, t)
    return int(t), tile_digest(img), [{k: int(s[k]) for k in STAT_KEYS} for s in st], time.perf_counter() - t0


def run_tiles(region, n: int, maxdwell: int, g: int, r: int, B: int, tiles: Sequence[int],
              procs: Optional[int] = None) -> Dict[int, dict]:
    """oracle.ask_tile for every listed tile, one process per core; {tile: record}."""
    import multiprocessing as mp
    build()
    procs = procs or len(os.sched_getaffinity(0))
    # longest first (big tiles near the set boundary dominate): a rough order by position is
    # not known in advance, so deal in the given order with chunksize 1
    jobs = [(tuple(region), n, maxdwell, g, r, B, int(t)) for t in tiles]
    out = {}
    if procs <= 1 or len(jobs) <= 1:
        res = [_one_tile(j) for j in jobs]
    else:
        with mp.get_context("fork").Pool(min(procs, len(jobs))) as pool:
            res = pool.map(_one_tile, jobs, chunksize=1)
    for t, sha, st, sec in res:
        out[t] = {"sha256": sha, "stats": st, "cpu_s": round(sec, 4)}
    return out


def _load(path: str, key_desc: dict) -> Optional[dict]:
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    return d if d.get("config") == key_desc else None


def tile_records(region, n: int, maxdwell: int, g: int, r: int, B: int, procs: Optional[int] = None,
                 store: bool = True) -> dict:
    """The oracle's per-tile digests and statistics for one whole configuration (all g*g
    tiles), from the golden files, the cache, or computed (then cached).  Returns
    {"config": ..., "tiles": {tile: {"sha256", "stats", "cpu_s"}}, "wall_s", "source"}."""
    key = config_key(region, n, maxdwell, g, r, B)
    desc = {"region": [float(v) for v in region], "n": int(n), "maxdwell": int(maxdwell), "g": int(g),
            "r": int(r), "B": int(B), "oracle_sha256": source_sha()}
    for src, d in (("golden", GOLDEN_DIR), ("cache", cache_dir())):
        rec = _load(os.path.join(d, key + ".json"), desc)
        if rec is not None:
            rec["tiles"] = {int(k): v for k, v in rec["tiles"].items()}
            rec["source"] = src
            return rec
    t0 = time.perf_counter()
    tiles = run_tiles(region, n, maxdwell, g, r, B, range(g * g), procs)
    rec = {"config": desc, "tiles": tiles, "wall_s": round(time.perf_counter() - t0, 3),
           "procs": procs or len(os.sched_getaffinity(0)), "source": "computed"}
    if store:
        os.makedirs(cache_dir(), exist_ok=True)
        save(rec, os.path.join(cache_dir(), key + ".json"))
    return rec


def save(rec: dict, path: str) -> None:
    tmp = path + f".tmp{os.getpid()}"
    body = {k: v for k, v in rec.items() if k != "source"}
    body["tiles"] = {str(k): v for k, v in sorted(rec["tiles"].items())}
    with open(tmp, "w") as f:
        json.dump(body, f, separators=(",", ":"))
    os.replace(tmp, path)


def summed_stats(rec: dict) -> List[dict]:
    """Per-level statistics of the whole image: the sum over the tiles' records."""
    out: List[dict] = []
    for t in rec["tiles"].values():
        for lv, s in enumerate(t["stats"]):
            while len(out) <= lv:
                out.append({k: 0 for k in STAT_KEYS})
            for k in STAT_KEYS:
                out[lv][k] += s[k]
    return out
