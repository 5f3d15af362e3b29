"""The tile-parallel oracle runner and its cache (oracle/cache.py) against the plain oracle:
digests equal those of the whole-image recursion's slices, the cache round-trips, and the
committed golden digests (tests/golden/oracle_tiles/, written by tools/make_oracle_golden.py)
belong to the CURRENT oracle source and agree with fresh oracle runs on sampled tiles."""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W
from oracle import cache


def test_run_tiles_digests_equal_whole_image_slices():
    w = W.Workload("c", W.NONDYADIC_REGIONS[0], 256, 800, 4, 2, 8)
    A, st = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    recs = cache.run_tiles(w.region, w.n, w.maxdwell, w.g, w.r, w.B, range(w.g * w.g), procs=4)
    d0 = w.n // w.g
    for t in range(w.g * w.g):
        gy, gx = divmod(t, w.g)
        assert recs[t]["sha256"] == cache.tile_digest(A[gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0]), t
    summed = cache.summed_stats({"tiles": recs})
    for a, b in zip(summed, st):
        for k in cache.STAT_KEYS:
            assert a[k] == b[k], k


def test_tile_records_cache_round_trip(tmp_path, monkeypatch):
    monkeypatch.setenv("ORACLE_CACHE_DIR", str(tmp_path))
    w = W.Workload("c", W.SEAHORSE_REGION, 128, 300, 4, 2, 4)
    a = cache.tile_records(w.region, w.n, w.maxdwell, w.g, w.r, w.B, procs=2)
    assert a["source"] == "computed"
    b = cache.tile_records(w.region, w.n, w.maxdwell, w.g, w.r, w.B, procs=2)
    assert b["source"] == "cache" and b["tiles"] == a["tiles"]
    # another maxdwell is another key
    c = cache.tile_records(w.region, w.n, w.maxdwell + 1, w.g, w.r, w.B, procs=2)
    assert c["source"] == "computed"


def _index():
    path = os.path.join(cache.GOLDEN_DIR, "index.json")
    return json.load(open(path))


def test_golden_digests_are_current():
    """Every committed golden file is keyed by the current oracle source: a change to
    oracle/*.c without re-running tools/make_oracle_golden.py fails here (the GPU tests would
    otherwise fall back to recomputing the oracle on the GPU box)."""
    idx = _index()
    names = {w.name: w for w in [W.C1, W.C3, W.C4, W.C5] + W.c2_sweep()}
    assert set(names) <= set(idx), sorted(set(names) - set(idx))
    for nm, w in names.items():
        key = cache.config_key(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
        assert idx[nm]["key"] == key, nm
        assert os.path.exists(os.path.join(cache.GOLDEN_DIR, key + ".json")), nm


def test_golden_c1_equals_whole_image_oracle():
    w = W.C1
    rec = cache.tile_records(w.region, w.n, w.maxdwell, w.g, w.r, w.B, store=False)
    assert rec["source"] == "golden"
    A, st = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    d0 = w.n // w.g
    for t, tr in rec["tiles"].items():
        gy, gx = divmod(t, w.g)
        assert tr["sha256"] == cache.tile_digest(A[gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0])
    for a, b in zip(cache.summed_stats(rec), st):
        assert all(a[k] == b[k] for k in cache.STAT_KEYS)


@pytest.mark.parametrize("name", ["C2_g8_r4_B16", "C2_g32_r2_B16", "C3", "C5"])
def test_golden_sampled_tiles_recomputed(name):
    """Two seeded random tiles of the configuration, recomputed now, equal the golden record."""
    w = {x.name: x for x in [W.C3, W.C5] + W.c2_sweep()}[name]
    rec = cache.tile_records(w.region, w.n, w.maxdwell, w.g, w.r, w.B, store=False)
    assert rec["source"] == "golden"
    rng = np.random.default_rng(W.SEED + len(name))
    for t in rng.choice(w.g * w.g, size=2, replace=False).tolist():
        img, st = oracle.ask_tile(w.region, w.n, w.maxdwell, w.g, w.r, w.B, t)
        assert cache.tile_digest(img) == rec["tiles"][t]["sha256"], t
        assert [{k: s[k] for k in cache.STAT_KEYS} for s in st] == rec["tiles"][t]["stats"], t
