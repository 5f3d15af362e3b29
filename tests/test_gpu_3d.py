"""GPU parity of the k = 3 ASK library (libmandel3d.so, NEXT-4) against the
3-D oracle (oracle/mandel3d_oracle.c), element by element, bit-exact."""
import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m3():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_02255_b200 import build
    build.build_3d()
    from paper_2206_02255_b200 import mandel3d
    return mandel3d


def _dec(st):
    return [{k: s[k] for k in ("regions_in", "filled", "subdivided", "leaves")} for s in st if s["regions_in"]]


@pytest.mark.parametrize("w", list(W.random_small_workloads3(24, seed=W.SEED + 61, max_n=64)), ids=lambda w: w.name)
def test_exhaustive3d_parity(m3, w):
    got = m3.exhaustive3d(w.region, w.n, w.maxdwell).cpu().numpy()
    assert np.array_equal(got, oracle.exhaustive3(w.region, w.n, w.maxdwell))


@pytest.mark.parametrize("flat", [False, True], ids=["refill", "flat"])
@pytest.mark.parametrize("w", list(W.random_small_workloads3(40, seed=W.SEED + 62, max_n=64)), ids=lambda w: w.name)
def test_ask3d_parity(m3, w, flat):
    ws = m3.workspace3d(w.n, w.g, w.r, w.B)
    got = m3.ask3d(w.region, w.n, w.maxdwell, w.g, w.r, w.B, ws=ws, stats=True, flat=flat).cpu().numpy()
    A, st = oracle.ask3(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    assert np.array_equal(got, A)
    gst = m3.ask3d_stats(ws)
    assert _dec(gst) == _dec(st)
    gl = [s for s in gst if s["regions_in"]]
    for lv, (a, b) in enumerate(zip(gl, st)):
        for k in ("leaf_px", "leaf_iters"):
            assert a[k] == b[k], (k, a, b)
        if lv == 0:  # level 0 computes whole surfaces, like the oracle
            assert a["border_px"] == b["border_px"] and a["border_iters"] == b["border_iters"]
        else:        # deeper levels reuse the parent's surface: only the division planes are new
            r, d = w.r, a["side"]
            new = (r * d - 2) ** 3 - (r * (d - 2)) ** 3
            assert a["border_px"] == gl[lv - 1]["subdivided"] * new
            assert a["border_iters"] <= b["border_iters"]


@pytest.mark.parametrize("n,g,r,B,md,region", [
    (128, 2, 2, 8, 300, W.DEFAULT_REGION3),     # 4 levels: 64, 32, 16, 8
    (128, 4, 4, 2, 200, W.DEFAULT_REGION3),     # r = 4, non-exact tiling: 32, 8, 2
    (64, 1, 2, 2, 150, (-0.875, -0.625, 0.0, 0.25, 0.0, 0.25)),
    (64, 32, 2, 2, 100, W.DEFAULT_REGION3),     # g * B == n: one level, 32768 regions
    (32, 2, 2, 4, 64, W.INTERIOR_REGION3),      # closed form: all maxdwell, 8 fills
    (32, 2, 2, 4, 64, W.ESCAPE_REGION3),        # closed form: all 1
    (64, 2, 2, 4, 1, W.DEFAULT_REGION3),        # maxdwell 1
    (64, 4, 2, 2, 333, (-2.25, -1.75, -0.25, 0.25, -0.5, 0.5)),  # |c| ~ 2: per-step voxels
])
def test_ask3d_edge_cases(m3, n, g, r, B, md, region):
    ws = m3.workspace3d(n, g, r, B)
    got = m3.ask3d(region, n, md, g, r, B, ws=ws).cpu().numpy()
    A, st = oracle.ask3(region, n, md, g, r, B)
    assert np.array_equal(got, A)
    assert _dec(m3.ask3d_stats(ws)) == _dec(st)
    ex = m3.exhaustive3d(region, n, md).cpu().numpy()
    assert np.array_equal(ex, oracle.exhaustive3(region, n, md))


@pytest.mark.parametrize("wname", ["V1", "V2"])
def test_full_size_3d_sampled_tiles(m3, wname):
    """The measured configurations at full size (tools/bench3d.py's launch): sampled level-0
    cubes equal the oracle's recursion on those cubes; sampled voxels of the exhaustive volume
    equal the oracle's dwell."""
    w = W.CONFIGS3[wname]
    ws = m3.workspace3d(w.n, w.g, w.r, w.B)
    vol = m3.ask3d(w.region, w.n, w.maxdwell, w.g, w.r, w.B, ws=ws)
    d0 = w.n // w.g
    rng = np.random.default_rng(W.SEED + 63)
    for t in rng.choice(w.g ** 3, size=2, replace=False).tolist():
        gx, gy, gz = t % w.g, (t // w.g) % w.g, t // (w.g * w.g)
        A, _ = oracle.ask3_tile(w.region, w.n, w.maxdwell, w.g, w.r, w.B, t)
        got = vol[gz * d0:(gz + 1) * d0, gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0].cpu().numpy()
        assert np.array_equal(got, A), t
    del vol
    ex = m3.exhaustive3d(w.region, w.n, w.maxdwell)
    for z in rng.integers(0, w.n, 2).tolist():
        assert np.array_equal(ex[z, :64].cpu().numpy(), oracle.exhaustive3(w.region, w.n, w.maxdwell, z, 1)[0, :64])


def test_shutdown_and_reuse(m3):
    """mandel3d_shutdown frees the fill stream/events; the next call recreates them."""
    from paper_2206_02255_b200 import _lib
    w = list(W.random_small_workloads3(1, seed=W.SEED + 64, max_n=32))[0]
    a = m3.ask3d(w.region, w.n, w.maxdwell, w.g, w.r, w.B).cpu().numpy()
    _lib.load_3d().mandel3d_shutdown()
    b = m3.ask3d(w.region, w.n, w.maxdwell, w.g, w.r, w.B).cpu().numpy()
    A, _ = oracle.ask3(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    assert np.array_equal(a, A) and np.array_equal(b, A)
