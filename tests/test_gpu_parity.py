"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element,
bit-exact (integer dwells).  Sizes span several tiles/levels and ragged cases; the full
BASELINE sizes are checked on sampled tiles/pixels the oracle computes one by one, in the
launch configuration bench.py times."""
import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SCHEMES = ("b200", "sbr", "mbr")


@pytest.fixture(scope="module")
def mb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2206_02255_b200 import build
    build.build()
    import paper_2206_02255_b200 as m
    return m


def _trim(stats):
    out = [s for s in stats if s["regions_in"] > 0]
    return out


def _cmp_stats(gpu, orc, scheme):
    gpu = _trim(gpu)
    assert len(gpu) == len(orc)
    for a, b in zip(gpu, orc):
        for k in ("regions_in", "filled", "subdivided", "leaves", "leaf_px", "leaf_iters"):
            assert a[k] == b[k], (k, a, b)
        if scheme in ("sbr", "mbr"):  # the paper's schemes recompute every region's full border
            assert a["border_px"] == b["border_px"] and a["border_iters"] == b["border_iters"]
        else:                # the B200 scheme computes each border pixel once
            assert a["border_px"] <= b["border_px"] and a["border_iters"] <= b["border_iters"]


# ----------------------------------------------------------------------------- exhaustive
@pytest.mark.parametrize("tuned", [False, True])
@pytest.mark.parametrize("w", [W.C1] + list(W.random_small_workloads(12, seed=W.SEED + 11, max_n=512)),
                         ids=lambda w: w.name)
def test_exhaustive_parity(mb, w, tuned):
    out = mb.exhaustive(w.region, w.n, w.maxdwell, tuned=tuned)
    E = oracle.exhaustive(w.region, w.n, w.maxdwell)
    assert np.array_equal(out.cpu().numpy(), E)


@pytest.mark.parametrize("tuned", [False, True])
@pytest.mark.parametrize("region", W.NONDYADIC_REGIONS)
def test_exhaustive_non_dyadic(mb, region, tuned):
    """Non-dyadic windows: the rounded pixel-centre mapping (R3) is bit-identical."""
    n, md = 512, 1200
    assert np.array_equal(mb.exhaustive(region, n, md, tuned=tuned).cpu().numpy(), oracle.exhaustive(region, n, md))


def test_exhaustive_pitched(mb):
    n = 128
    buf = torch.full((n, n + 37), -7, dtype=torch.int32, device="cuda")  # row pitch n + 37
    mb.exhaustive(W.SEAHORSE_REGION, n, 900, out=buf)
    E = oracle.exhaustive(W.SEAHORSE_REGION, n, 900)
    got = buf.cpu().numpy()
    assert np.array_equal(got[:, :n], E)
    assert np.all(got[:, n:] == -7)


# ----------------------------------------------------------------------------- ASK
@pytest.mark.parametrize("scheme", SCHEMES)
def test_ask_c1(mb, scheme):
    w = W.C1
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    out = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, ws=ws, scheme=scheme, stats=True)
    A, st = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    assert np.array_equal(out.cpu().numpy(), A)
    _cmp_stats(mb.ask_stats(ws), st, scheme)


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("w", list(W.random_small_workloads(30, seed=W.SEED + 12, max_n=512)),
                         ids=lambda w: w.name)
def test_ask_random_small(mb, w, scheme):
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    out = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, ws=ws, scheme=scheme, stats=True)
    A, st = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    assert np.array_equal(out.cpu().numpy(), A)
    _cmp_stats(mb.ask_stats(ws), st, scheme)


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("n,g,r,B,md,region", [
    (256, 2, 2, 2, 300, W.DEFAULT_REGION),      # smallest leaves (side 2: empty interior)
    (512, 4, 8, 2, 500, W.SEAHORSE_REGION),     # r = 8, leaf side 2..15
    (1024, 2, 4, 32, 700, W.DEFAULT_REGION),    # non-exact tiling: 512,128,32
    (2048, 2, 8, 16, 256, W.DEFAULT_REGION),    # non-exact: 1024,128,16
    (256, 128, 2, 2, 100, W.DEFAULT_REGION),    # g*B == n: single level, 16384 tiles
    (512, 1, 2, 4, 1000, W.SEAHORSE_REGION),    # g = 1: one level-0 region
    (256, 4, 2, 8, 1, W.DEFAULT_REGION),        # maxdwell 1: everything uniform
    (256, 4, 2, 8, 64, W.INTERIOR_REGION),      # closed form: all maxdwell
    (256, 4, 2, 8, 64, W.ESCAPE_REGION),        # closed form: all 1
    (2048, 8, 2, 16, 3000, (-0.75, -0.5, 0.0, 0.25)),  # maxdwell not a multiple of the chunk
    (1024, 8, 2, 16, 2000, W.NONDYADIC_REGIONS[0]),    # non-dyadic windows: rounded
    (512, 4, 4, 8, 700, W.NONDYADIC_REGIONS[1]),       # pixel centres, op order decides bits
    (256, 2, 2, 4, 1500, W.NONDYADIC_REGIONS[2]),      # non-square window (dx != dy)
])
def test_ask_edge_cases(mb, scheme, n, g, r, B, md, region):
    ws = mb.workspace(n, g, r, B)
    out = mb.ask(region, n, md, g, r, B, ws=ws, scheme=scheme, stats=True)
    A, st = oracle.ask(region, n, md, g, r, B)
    assert np.array_equal(out.cpu().numpy(), A)
    _cmp_stats(mb.ask_stats(ws), st, scheme)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_ask_tiles_subset_and_pitch(mb, scheme):
    n, g, r, B, md = 512, 8, 2, 8, 800
    rng = np.random.default_rng(W.SEED)
    tiles = rng.permutation(g * g)[:23].tolist()
    buf = torch.full((n, n + 4), -5, dtype=torch.int32, device="cuda")  # pitch n+4 (vector path)
    ws = mb.workspace(n, g, r, B)
    mb.ask(W.SEAHORSE_REGION, n, md, g, r, B, out=buf, ws=ws, tiles=tiles, scheme=scheme, stats=True)
    A, st = oracle.ask(W.SEAHORSE_REGION, n, md, g, r, B, tiles=tiles)
    got = buf.cpu().numpy()
    mine = A != -1                                   # pixels of the listed tiles
    assert mine.sum() == len(tiles) * (n // g) ** 2
    assert np.array_equal(got[:, :n][mine], A[mine])
    assert np.all(got[:, :n][~mine] == -5) and np.all(got[:, n:] == -5)
    _cmp_stats(mb.ask_stats(ws), st, scheme)


def test_ask_unaligned_pitch_scalar_fill(mb):
    n, g, r, B, md = 256, 4, 2, 8, 500
    buf = torch.full((n, n + 3), -1, dtype=torch.int32, device="cuda")
    mb.ask(W.DEFAULT_REGION, n, md, g, r, B, out=buf)
    A, _ = oracle.ask(W.DEFAULT_REGION, n, md, g, r, B)
    assert np.array_equal(buf.cpu().numpy()[:, :n], A)


def test_ask_equals_lookup_of_gpu_exhaustive(mb):
    """mandel_ask == ask_by_lookup(mandel_exhaustive), on the seahorse window."""
    n, g, r, B, md = 2048, 16, 4, 8, 2048
    E = mb.exhaustive(W.SEAHORSE_REGION, n, md).cpu().numpy()
    A = mb.ask(W.SEAHORSE_REGION, n, md, g, r, B).cpu().numpy()
    L, _ = oracle.ask_by_lookup(E, g, r, B)
    assert np.array_equal(A, L)


def test_repeat_calls_reuse_graph_and_are_deterministic(mb):
    w = W.C1
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
    a = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws).clone()
    c0 = mb.graph_captures()
    for _ in range(3):
        b = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws)
        assert torch.equal(a, b)
    # a different region through the same workspace/output: same graph, oracle's image
    b = mb.ask(W.SEAHORSE_REGION, w.n, w.maxdwell, w.g, w.r, w.B, out=out, ws=ws)
    A, _ = oracle.ask(W.SEAHORSE_REGION, w.n, w.maxdwell, w.g, w.r, w.B)
    assert np.array_equal(b.cpu().numpy(), A)
    assert mb.graph_captures() == c0


def test_one_graph_serves_views_maxdwell_and_tile_lists(mb):
    """Device-side parameter block: three different views,
    maxdwell values and tile lists of the same size run through ONE captured graph, each
    bit-exact against the oracle; the first call's capture + instantiate cost is reported."""
    import time
    n, g, r, B = 512, 8, 2, 8
    ws = mb.workspace(n, g, r, B)
    out = torch.empty((n, n), dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(W.SEED + 77)
    cases = [(W.SEAHORSE_REGION, 900), ((-0.74531, -0.74419, 0.11273, 0.11385), 1500),
             (W.DEFAULT_REGION, 300)]
    c0 = mb.graph_captures()
    times = []
    for i, (region, md) in enumerate(cases):
        tiles = rng.permutation(g * g)[:21].tolist()
        out.fill_(-9)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mb.ask(region, n, md, g, r, B, out=out, ws=ws, tiles=tiles)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        A, _ = oracle.ask(region, n, md, g, r, B, tiles=tiles)
        got = out.cpu().numpy()
        mine = A != -1
        assert np.array_equal(got[mine], A[mine]), i
        assert np.all(got[~mine] == -9), i
        assert mb.graph_captures() == c0 + 1, i   # captured by the first call only
    print(f"first call (capture + instantiate + run) {1e3 * times[0]:.2f} ms, "
          f"later calls {1e3 * times[1]:.2f} / {1e3 * times[2]:.2f} ms")


def test_ask_to_host(mb):
    w = W.C1
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    out = torch.empty((w.n, w.n), dtype=torch.int32, device="cuda")
    h = torch.empty(w.n * w.n, dtype=torch.int32).pin_memory()
    mb.ask_to_host(w.region, w.n, w.maxdwell, w.g, w.r, w.B, h, out, ws)
    A, _ = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    assert np.array_equal(h.numpy().reshape(w.n, w.n), A)


@pytest.mark.parametrize("n,g,r,B,md", [(2048, 16, 2, 16, 700), (1024, 2, 4, 8, 300), (512, 8, 8, 4, 900)])
def test_ask_to_host_banded(mb, n, g, r, B, md):
    """The whole-image host call is pipelined over bands of tile rows (copy of one band
    overlapping the next band's ASK): the host image equals the oracle's, every pixel, also
    with a pitched device buffer."""
    ws = mb.workspace(n, g, r, B)
    out = torch.full((n, n + 4), -3, dtype=torch.int32, device="cuda")
    h = torch.full((n * n,), -7, dtype=torch.int32).pin_memory()
    mb.ask_to_host(W.SEAHORSE_REGION, n, md, g, r, B, h, out, ws)
    A, _ = oracle.ask(W.SEAHORSE_REGION, n, md, g, r, B)
    assert np.array_equal(h.numpy().reshape(n, n), A)


@pytest.mark.parametrize("n,g,r,B,md,pad", [(2048, 16, 2, 16, 700, 4), (1024, 2, 4, 8, 300, 0),
                                            (512, 8, 8, 4, 900, 3), (256, 4, 2, 8, 65535, 0)])
def test_ask_to_host_u16(mb, n, g, r, B, md, pad):
    """The 16-bit host image (mandel_ask_to_host_u16): every pixel equals the oracle's dwell,
    for the banded whole image and for a tile subset, with pitched device buffers (scalar
    narrowing path) and unpitched ones (vector path), up to maxdwell 65535."""
    ws = mb.workspace(n, g, r, B)
    out = torch.full((n, n + pad), -3, dtype=torch.int32, device="cuda")
    stage = torch.full((n * n,), -1, dtype=torch.int16, device="cuda")
    h = torch.full((n * n,), 7, dtype=torch.uint16).pin_memory()
    mb.ask_to_host(W.SEAHORSE_REGION, n, md, g, r, B, h, out, ws, stage=stage)
    A, _ = oracle.ask(W.SEAHORSE_REGION, n, md, g, r, B)
    assert np.array_equal(h.numpy().reshape(n, n).astype(np.int64), A)
    tiles = _sample_tiles(g, max(1, g * g // 3), seed=5)
    h2 = torch.zeros((n * n,), dtype=torch.uint16).pin_memory()
    mb.ask_to_host(W.SEAHORSE_REGION, n, md, g, r, B, h2, out, ws, tiles=tiles)
    got = h2.numpy().reshape(n, n).astype(np.int64)
    d0 = n // g
    for t in range(g * g):
        ty, tx = divmod(t, g)
        sl = (slice(ty * d0, (ty + 1) * d0), slice(tx * d0, (tx + 1) * d0))
        if t in tiles:
            assert np.array_equal(got[sl], A[sl]), t
        else:
            assert not got[sl].any(), t


def test_ask_to_host_u16_rejects(mb):
    """maxdwell > 65535 does not fit the 16-bit image: MANDEL_EINVAL, nothing written."""
    n, g, r, B = 128, 2, 2, 8
    ws = mb.workspace(n, g, r, B)
    out = torch.empty((n, n), dtype=torch.int32, device="cuda")
    h = torch.zeros((n * n,), dtype=torch.uint16)
    with pytest.raises(Exception):
        mb.ask_to_host(W.DEFAULT_REGION, n, 65536, g, r, B, h, out, ws)
    assert not h.numpy().any()


# ----------------------------------------------------------------------------- full sizes
def _sample_tiles(g, k, seed):
    rng = np.random.default_rng(seed)
    return sorted(rng.choice(g * g, size=k, replace=False).tolist())


@pytest.mark.parametrize("wname", ["C3", "C5", "C4"])
def test_full_size_ask_sampled_tiles(mb, wname):
    """BASELINE C3 / C5 at full size in bench.py's launch configuration (all g*g tiles, B200
    scheme): sampled level-0 tiles equal the oracle's recursion on those tiles."""
    w = W.CONFIGS[wname]
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    out = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, ws=ws, stats=True)
    torch.cuda.synchronize()
    st = mb.ask_stats(ws)
    # bench.py's timed launch (no counters, PDL chain, events around the leaf kernel) gives the
    # same image
    bench_img = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, ws=ws, timing="leaf")
    torch.cuda.synchronize()
    assert torch.equal(bench_img, out)
    del bench_img
    d0 = w.n // w.g
    tiles = _sample_tiles(w.g, 2 if wname == "C4" else 3, W.SEED + int(wname[1]))
    for t in tiles:
        gy, gx = divmod(t, w.g)
        A, _ = oracle.ask_tile(w.region, w.n, w.maxdwell, w.g, w.r, w.B, t)
        got = out[gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0].cpu().numpy()
        assert np.array_equal(got, A), t
    # structural identities at full size
    st = _trim(st)
    for a, b in zip(st, st[1:]):
        assert b["regions_in"] == w.r * w.r * a["subdivided"]
    for s in st:
        assert s["regions_in"] == s["filled"] + s["subdivided"] + s["leaves"]


@pytest.mark.parametrize("wname", ["C3", "C5", "C4"])
def test_full_size_exhaustive_sampled_pixels(mb, wname):
    w = W.CONFIGS[wname]
    out = mb.exhaustive(w.region, w.n, w.maxdwell, tuned=True)
    # the tuned kernel's image equals the plain one's on every pixel
    plain = mb.exhaustive(w.region, w.n, w.maxdwell)
    torch.cuda.synchronize()
    assert torch.equal(out, plain)
    del plain
    rng = np.random.default_rng(W.SEED)
    ii = rng.integers(0, w.n, 4000)
    jj = rng.integers(0, w.n, 4000)
    ref = oracle.dwell_pixels(w.region, w.n, w.maxdwell, ii, jj)
    got = out[torch.as_tensor(ii, device="cuda"), torch.as_tensor(jj, device="cuda")].cpu().numpy()
    assert np.array_equal(got, ref)
    # plus two full rows (a ragged mix of inside / outside)
    for i in (w.n // 2 - 1, w.n // 3):
        assert np.array_equal(out[i].cpu().numpy(), oracle.exhaustive(w.region, w.n, w.maxdwell, i, 1)[0])


@pytest.mark.parametrize("md", [1, 2, 3, 7, 8, 9, 15, 16, 17, 31, 32, 33, 63, 65, 100, 257])
def test_ask_maxdwell_not_multiple_of_chunk(mb, md):
    """The lane-refill kernels run K-step chunks and find the exact dwell by bisection over
    the last chunk, capped at maxdwell: maxdwell values around multiples of K (8, 16, 32)."""
    n, g, r, B = 256, 4, 2, 8
    for region in (W.DEFAULT_REGION, W.SEAHORSE_REGION):
        ws = mb.workspace(n, g, r, B)
        out = mb.ask(region, n, md, g, r, B, ws=ws)
        A, _ = oracle.ask(region, n, md, g, r, B)
        assert np.array_equal(out.cpu().numpy(), A), (region, md)
        ex = mb.exhaustive(region, n, md).cpu().numpy()
        assert np.array_equal(ex, oracle.exhaustive(region, n, md)), (region, md)
        ext = mb.exhaustive(region, n, md, tuned=True).cpu().numpy()
        assert np.array_equal(ext, ex), (region, md)


def test_ask_large_region_outside_radius(mb):
    """|c|^2 > 3.9 pixels take the per-step path (escape permanence is not guaranteed
    there): a window straddling |c| = 2 on the negative real axis, including c = -2."""
    region = (-2.25, -1.75, -0.25, 0.25)
    n, g, r, B, md = 256, 2, 2, 8, 700
    out = mb.ask(region, n, md, g, r, B)
    A, _ = oracle.ask(region, n, md, g, r, B)
    assert np.array_equal(out.cpu().numpy(), A)


@pytest.mark.parametrize("flags", [dict(flat=True), dict(serial=True), dict(flat=True, serial=True)])
@pytest.mark.parametrize("w", [W.C1, W.Workload("sea2k", W.SEAHORSE_REGION, 2048, 1500, 8, 4, 16)],
                         ids=lambda w: w.name if hasattr(w, "name") else str(w))
def test_ask_ab_variants(mb, w, flags):
    """The A/B variants (plain thread-per-pixel kernels, fills on the main stream) produce
    the same image as the oracle too."""
    out = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, **flags)
    A, _ = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    assert np.array_equal(out.cpu().numpy(), A)


@pytest.mark.parametrize("groups", [2, 3, 8])
def test_ask_groups(mb, groups):
    """Independent ASK chains over round-robin tile subsets (MANDEL_FLAG_GROUPS): same image
    and the same summed level statistics as the oracle, with and without a tile subset."""
    w = W.Workload("g", W.SEAHORSE_REGION, 1024, 900, 8, 2, 16)
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    out = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, ws=ws, groups=groups, stats=True)
    A, st = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    assert np.array_equal(out.cpu().numpy(), A)
    _cmp_stats(mb.ask_stats(ws), st, "b200")
    tiles = [5, 17, 2, 40, 63, 33, 9]
    buf = torch.full((w.n, w.n), -3, dtype=torch.int32, device="cuda")
    mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, out=buf, ws=ws, tiles=tiles, groups=groups, stats=True)
    At, stt = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, tiles=tiles)
    mine = At != -1
    assert np.array_equal(buf.cpu().numpy()[mine], At[mine]) and np.all(buf.cpu().numpy()[~mine] == -3)
    _cmp_stats(mb.ask_stats(ws), stt, "b200")


# ----------------------------------------------------------------------------- DP baseline
# libmandel_dp.so (include/mandel_dp.h): recursive Dynamic Parallelism, same decisions per
# region as ASK, hence the same image as the oracle's ASK recursion.
@pytest.mark.parametrize("w", [W.C1] + list(W.random_small_workloads(12, seed=W.SEED + 21, max_n=512)),
                         ids=lambda w: w.name)
def test_dp_parity(mb, w):
    out = mb.dp(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    A, _ = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    assert np.array_equal(out.cpu().numpy(), A)


@pytest.mark.parametrize("n,g,r,B,md,region", [
    (1024, 2, 4, 32, 700, W.DEFAULT_REGION),    # non-exact tiling
    (512, 1, 2, 4, 1000, W.SEAHORSE_REGION),    # g = 1, 8 levels of recursion
    (256, 4, 2, 8, 64, W.INTERIOR_REGION),      # closed form: all maxdwell (no launches)
])
def test_dp_edge_cases(mb, n, g, r, B, md, region):
    buf = torch.full((n, n + 3), -1, dtype=torch.int32, device="cuda")  # unaligned pitch: scalar fill
    mb.dp(region, n, md, g, r, B, out=buf)
    A, _ = oracle.ask(region, n, md, g, r, B)
    got = buf.cpu().numpy()
    assert np.array_equal(got[:, :n], A) and np.all(got[:, n:] == -1)


def test_dp_full_size_c3_equals_ask(mb):
    """C3 at full size: the DP tree's image equals mandel_ask's (bit-exact, every pixel), and
    sampled tiles equal the oracle."""
    w = W.C3
    a = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    d = mb.dp(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    torch.cuda.synchronize()
    assert torch.equal(a, d)
    d0 = w.n // w.g
    t = _sample_tiles(w.g, 1, W.SEED + 31)[0]
    gy, gx = divmod(t, w.g)
    A, _ = oracle.ask_tile(w.region, w.n, w.maxdwell, w.g, w.r, w.B, t)
    assert np.array_equal(d[gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0].cpu().numpy(), A)


# ----------------------------------------------------------------------------- tile costs
@pytest.mark.parametrize("n,g,r,B,md,region", [
    (256, 4, 2, 8, 500, W.DEFAULT_REGION),
    (512, 8, 2, 16, 900, W.SEAHORSE_REGION),
    (256, 16, 2, 4, 300, W.DEFAULT_REGION),
])
def test_tile_costs_match_oracle(mb, n, g, r, B, md, region):
    """MANDEL_FLAG_TILE_COST (the multi-GPU deal's per-tile cost): for the B200 scheme every
    pixel is computed once unless it lies strictly inside a filled region, so a tile's executed
    iterations are the exhaustive dwells of its pixels minus those of its filled regions'
    interiors (oracle terminal-region records; independent of the GPU path)."""
    ws = mb.workspace(n, g, r, B)
    mb.ask(region, n, md, g, r, B, ws=ws, tile_cost=True)
    got = mb.tile_costs(ws, g)
    E = oracle.exhaustive(region, n, md).astype(np.int64)
    _, _, recs = oracle.ask(region, n, md, g, r, B, want_regions=True)
    inner = np.zeros((n, n), dtype=bool)
    for x, y, d, kind, _v, _l in recs.tolist():
        if kind == 0 and d > 2:
            inner[y + 1:y + d - 1, x + 1:x + d - 1] = True
    d0 = n // g
    want = [int(E[gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0][~inner[gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0]].sum())
            for gy in range(g) for gx in range(g)]
    assert got == want


@pytest.mark.parametrize("n,g,r,B,md,region", [
    (256, 4, 2, 8, 500, W.DEFAULT_REGION),
    (512, 8, 2, 16, 900, W.SEAHORSE_REGION),
    (1024, 16, 4, 8, 700, W.NONDYADIC_REGIONS[0]),
])
def test_tile_costs_sampled_match_oracle(mb, n, g, r, B, md, region):
    """MANDEL_FLAG_TILE_COST_SAMPLED (the multi-GPU deal's per-step feedback): the same pixel
    set as the exact counters, but only pixels with (x + y) % 64 == 0, each counted as
    64 * (dwell + 64) (iterations plus the per-pixel work, ask_kernels.cuh TC_PX_COST) -- an
    exact identity against the oracle; the image is unchanged; and the estimate is close to
    the same cost summed over every computed pixel (checked loosely: a 1/64 lattice sample)."""
    ws = mb.workspace(n, g, r, B)
    out = mb.ask(region, n, md, g, r, B, ws=ws, tile_cost="sampled")
    got = mb.tile_costs(ws, g)
    A, _, recs = oracle.ask(region, n, md, g, r, B, want_regions=True)
    assert np.array_equal(out.cpu().numpy(), A)
    E = oracle.exhaustive(region, n, md).astype(np.int64)
    inner = np.zeros((n, n), dtype=bool)
    for x, y, d, kind, _v, _l in recs.tolist():
        if kind == 0 and d > 2:
            inner[y + 1:y + d - 1, x + 1:x + d - 1] = True
    yy, xx = np.indices((n, n))
    lattice = (xx + yy) % 64 == 0
    d0 = n // g
    sl = lambda M, gy, gx: M[gy * d0:(gy + 1) * d0, gx * d0:(gx + 1) * d0]  # noqa: E731
    K = 64  # TC_PX_COST
    want = [64 * int((sl(E, gy, gx)[~sl(inner, gy, gx) & sl(lattice, gy, gx)] + K).sum())
            for gy in range(g) for gx in range(g)]
    assert got == want
    exact = [int((sl(E, gy, gx)[~sl(inner, gy, gx)] + K).sum()) for gy in range(g) for gx in range(g)]
    assert abs(sum(got) - sum(exact)) <= 0.1 * sum(exact)


def test_device_plan_frame_loop(mb):
    """DevicePlan.step, bench.py's N > 1 frame loop with the one-step-lagged side-stream plan,
    run for every rank of a P-way deal on one GPU: each frame the ranks together render the
    oracle's image (no tile twice, none missing) and from the third frame on the partition is
    the LPT deal of the sampled costs."""
    from paper_2206_02255_b200 import deal, multigpu
    w = W.Workload("fl", W.DEFAULT_REGION, 1024, 1000, 16, 2, 16)
    A, _ = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    P = 4
    plans = [multigpu.DevicePlan(w, P, r, torch.device("cuda"), sample_every=1) for r in range(P)]
    c0 = torch.zeros(w.g * w.g, dtype=torch.int64, device="cuda")
    plans[0].preview_costs(c0)
    for p in plans:
        p.deal(c0, both=True)
    wss = [mb.workspace(w.n, w.g, w.r, w.B) for _ in range(P)]
    out = torch.full((w.n, w.n), -1, dtype=torch.int32, device="cuda")
    for frame in range(4):
        out.fill_(-1)
        lists = [p.host_tiles() for p in plans]
        assert sorted(k for l in lists for k in l) == list(range(w.g * w.g)), frame
        views = []
        for p, ws in zip(plans, wss):
            p.step(out, ws, lambda t: views.append(t))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), A), frame
        # the side streams dealt on each rank's own counters; redo it on what the NCCL
        # all-reduce would have left in every rank's buffer: the sum over the ranks
        total = sum(views)
        for v in views:
            v.copy_(total)
        for p in plans:
            k = 1 - p.cur
            mb.deal_lpt(p.cbuf2[k], P, p.rank, p.tiles2[k], p.count2[k])
        torch.cuda.synchronize()
        want = deal.lpt(total.tolist(), P)
        for p in plans:
            k = 1 - p.cur
            assert p.tiles2[k][: int(p.count2[k].item())].tolist() == want[p.rank]


def test_device_plan_sampling_period(mb):
    """The default frame loop counts and re-deals only every SAMPLE_EVERY-th frame (odd, so
    both alternating lists are re-dealt): every frame's image is the oracle's, the partition is
    complete every frame, the counters are all-reduced on the same frames on every rank, and
    both lists end up dealt on the sampled costs."""
    from paper_2206_02255_b200 import deal, multigpu
    w = W.Workload("fs", W.SEAHORSE_REGION, 1024, 900, 16, 2, 16)
    A, _ = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    P, E = 3, multigpu.SAMPLE_EVERY
    assert E % 2 == 1
    plans = [multigpu.DevicePlan(w, P, r, torch.device("cuda")) for r in range(P)]
    c0 = torch.zeros(w.g * w.g, dtype=torch.int64, device="cuda")
    plans[0].preview_costs(c0)
    for p in plans:
        p.deal(c0, both=True)
    wss = [mb.workspace(w.n, w.g, w.r, w.B) for _ in range(P)]
    out = torch.full((w.n, w.n), -1, dtype=torch.int32, device="cuda")
    calls = []
    for frame in range(2 * E + 1):
        out.fill_(-1)
        lists = [p.host_tiles() for p in plans]
        assert sorted(k for l in lists for k in l) == list(range(w.g * w.g)), frame
        views = []
        for p, ws in zip(plans, wss):
            p.step(out, ws, lambda t: views.append(t))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), A), frame
        assert len(views) in (0, P), frame
        calls.append(len(views) > 0)
        if views:  # what the all-reduce would leave: re-deal both ranks' lists on the sum
            total = sum(views)
            for v in views:
                v.copy_(total)
            for p in plans:
                k = 1 - p.cur
                mb.deal_lpt(p.cbuf2[k], P, p.rank, p.tiles2[k], p.count2[k])
            torch.cuda.synchronize()
    assert calls == [f % E == 0 for f in range(2 * E + 1)]


def test_timing_modes(mb):
    """bench.py's timed steps use MANDEL_FLAG_TIMING_LEAF: events around the leaf kernel only
    (the level chain keeps its programmatic-dependent-launch edges); MANDEL_FLAG_TIMING times
    every kernel.  Both leave the image unchanged."""
    w = W.C1
    ws = mb.workspace(w.n, w.g, w.r, w.B)
    A, _ = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    out = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, ws=ws, timing="leaf")
    kt = mb.kernel_times()
    assert [k["kind"] for k in kt] == ["b200_leaf"] and kt[0]["ms"] > 0
    assert np.array_equal(out.cpu().numpy(), A)
    out = mb.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B, ws=ws, timing=True)
    kinds = [k["kind"] for k in mb.kernel_times()]
    L = mb.levels(w.n, w.g, w.r, w.B)
    assert kinds.count("b200_border") == L and kinds.count("b200_classify") == L
    assert kinds.count("fill") == L and kinds.count("b200_leaf") == 1 and kinds[0] == "init"
    assert np.array_equal(out.cpu().numpy(), A)


@pytest.mark.parametrize("scheme", ["b200", "sbr", "mbr"])
def test_ask_empty_tile_subset(mb, scheme):
    """A rank can receive no level-0 tile (more ranks than tiles): an empty subset writes
    nothing, reports zero regions, and the workspace serves a full call afterwards."""
    n, g, r, B, md = 128, 2, 2, 8, 300
    ws = mb.workspace(n, g, r, B)
    buf = torch.full((n, n), -5, dtype=torch.int32, device="cuda")
    mb.ask(W.DEFAULT_REGION, n, md, g, r, B, out=buf, ws=ws, tiles=[], scheme=scheme, stats=True)
    torch.cuda.synchronize()
    assert int((buf != -5).sum().item()) == 0
    assert all(s["regions_in"] == 0 and s["filled"] == 0 for s in mb.ask_stats(ws))
    h = torch.full((n * n,), -5, dtype=torch.int32).pin_memory()
    mb.ask_to_host(W.DEFAULT_REGION, n, md, g, r, B, h, buf, ws, tiles=[], scheme=scheme)
    assert int((h != -5).sum().item()) == 0
    A, _ = oracle.ask(W.DEFAULT_REGION, n, md, g, r, B)
    assert np.array_equal(mb.ask(W.DEFAULT_REGION, n, md, g, r, B, ws=ws, scheme=scheme).cpu().numpy(), A)


@pytest.mark.parametrize("md", [65537, 200003])
def test_large_maxdwell(mb, md):
    """maxdwell beyond 2^16 and not a multiple of any chunk: the closed-form interior window is
    all maxdwell for Ex and every scheme; a boundary window matches the oracle."""
    n, g, r, B = 32, 2, 2, 4
    for scheme in ("b200", "sbr", "mbr"):
        out = mb.ask(W.INTERIOR_REGION, n, md, g, r, B, scheme=scheme).cpu().numpy()
        assert np.all(out == md), scheme
    assert np.all(mb.exhaustive(W.INTERIOR_REGION, n, md).cpu().numpy() == md)
    assert np.all(mb.exhaustive(W.INTERIOR_REGION, n, md, tuned=True).cpu().numpy() == md)
    region = (-0.75, -0.734375, 0.09375, 0.109375)  # seahorse boundary, dyadic
    A, _ = oracle.ask(region, 16, md, 2, 2, 4)
    assert np.array_equal(mb.ask(region, 16, md, 2, 2, 4).cpu().numpy(), A)
    assert np.array_equal(mb.exhaustive(region, 16, md).cpu().numpy(), oracle.exhaustive(region, 16, md))


# ----------------------------------------------------------------------------- device deal
@pytest.mark.parametrize("G,world", [(256, 8), (256, 3), (64, 8), (16, 5), (4096, 8), (1, 1)])
def test_device_lpt_equals_host_lpt(mb, G, world):
    """mandel_deal_lpt (one block: bitonic sort + greedy list schedule) gives every rank exactly
    the host LPT deal (paper_2206_02255_b200.deal.lpt), ties included."""
    from paper_2206_02255_b200 import deal
    rng = np.random.default_rng(W.SEED + G + world)
    costs = (rng.pareto(1.3, G) * 1e6).astype(np.int64)
    costs[rng.choice(G, size=min(G, 7), replace=False)] = 12345  # ties
    want = deal.lpt(costs.tolist(), world)
    dc = torch.as_tensor(costs, device="cuda")
    for rank in range(world):
        t = torch.full((G,), -1, dtype=torch.int32, device="cuda")
        c = torch.zeros(1, dtype=torch.int32, device="cuda")
        mb.deal_lpt(dc, world, rank, t, c)
        assert t[: int(c.item())].tolist() == want[rank], rank


def test_ask_device_tile_list_and_device_plan(mb):
    """mandel_ask_dtiles: the tile list is read on the device when the call runs -- a deal kernel
    on the same stream chooses it -- and one graph serves every list; the ranks of a P-way
    device plan together produce the oracle's image (no tile twice, none missing)."""
    from paper_2206_02255_b200 import multigpu
    w = W.Workload("dt", W.SEAHORSE_REGION, 512, 900, 8, 2, 8)
    A, _ = oracle.ask(w.region, w.n, w.maxdwell, w.g, w.r, w.B)
    out = torch.full((w.n, w.n), -1, dtype=torch.int32, device="cuda")
    costs = torch.zeros(w.g * w.g, dtype=torch.int64, device="cuda")
    P = 3
    plans = [multigpu.DevicePlan(w, P, r, torch.device("cuda")) for r in range(P)]
    plans[0].preview_costs(costs)
    seen = []
    wss = [mb.workspace(w.n, w.g, w.r, w.B) for _ in range(P)]
    for step in range(2):
        for p in plans:
            p.deal(costs)
        out.fill_(-1)
        c0 = mb.graph_captures()
        for p, ws in zip(plans, wss):
            p.render(out, ws)
            seen += p.host_tiles()
        if step == 1:
            assert mb.graph_captures() == c0  # same graphs as step 0, new device lists
        assert np.array_equal(out.cpu().numpy(), A), step
        costs.zero_()
        for ws in wss:
            costs += mb.tile_cost_view(ws, w.n, w.g, w.r, w.B)
    assert sorted(seen[: w.g * w.g]) == list(range(w.g * w.g))
