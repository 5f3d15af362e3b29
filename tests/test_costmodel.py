"""Cost model pinned to SPEC.md's worked examples, closed forms at P in {0, 1},
the paper's stated bounds (Omega <= A, S <= A) and a Monte-Carlo simulation of the
subdivision tree (oracle/montecarlo.py)."""
import math
import os

import numpy as np
import pytest

from oracle import montecarlo
from paper_2206_02255_b200 import costmodel as cm

import workloads as W


def test_depth_tau_spec_examples():
    # SPEC.md S:47-51
    assert cm.depth_tau(65536, 16, 2, 32) == 7
    assert cm.depth_tau(256, 2, 2, 128) == 1
    assert cm.depth_tau(1024, 4, 4, 16) == 2
    # the built ASK runs one more level (leaf side B)
    assert cm.depth_tau(1024, 4, 2, 32, "leaf") == 4  # C1: 256,128,64,32
    with pytest.raises(ValueError):
        cm.depth_tau(64, 8, 2, 16)


def test_exhaustive_work_and_time_spec_examples():
    assert cm.exhaustive_work(4, 1) == 16
    assert cm.exhaustive_work(1024, 512) == 536870912
    assert cm.exhaustive_time(1024, 128, 64, 512) == 65536
    assert cm.exhaustive_time(8, 128, 64, 1) == 1
    assert cm.exhaustive_time(65536, 128, 64, 512) == 268435456


def test_ssd_work_closed_forms():
    # tau = 1: empty sum, W = n^2 A
    p = cm.ModelParams(256, 2, 2, 128, P=0.3, A=512)
    assert cm.ssd_work(p) == 256 * 256 * 512
    assert cm.work_reduction_factor(p) == 1.0
    # P = 0, tau >= 2: W = 4 n g A + n^2, Omega ~= 56.89
    p = cm.ModelParams(1024, 4, 2, 16, P=0.0, A=512)
    assert cm.depth_tau(1024, 4, 2, 16) >= 2
    assert cm.ssd_work(p) == 4 * 1024 * 4 * 512 + 1024 ** 2 == 9437184
    assert abs(cm.work_reduction_factor(p) - 56.8889) < 1e-3
    # P = 1: every region subdivides, nothing terminates: W = sum_i Q_i G R^i + lam A G R^i + n^2 A
    n, g, r, B, A, lam = 4096, 16, 2, 32, 512, 10
    p = cm.ModelParams(n, g, r, B, P=1.0, A=A, lam=lam)
    tau = cm.depth_tau(n, g, r, B)
    expect = sum((4 * n * A / (g * r ** i) + lam * A) * g * g * r ** (2 * i) for i in range(tau - 1)) + n * n * A
    assert math.isclose(cm.ssd_work(p), expect, rel_tol=1e-12)


def test_general_equals_ssd_for_constant_P():
    """Eq. general with constant P and the Mandelbrot Q/T levels equals W^M_SSD; the
    general form with level-independent Q,S,T at tau=1 reduces to n^2 A."""
    assert cm.general_subdivision_work(64, 2, 2, 1, [], 10, 2, 16, 4) == 64 * 64 * 4
    assert cm.general_subdivision_work(64, 2, 2, 2, [0.0], 10, 2, 16, 4) == 4 * (10 + 16)


@pytest.mark.parametrize("P", [0.0, 1.0])
def test_montecarlo_exact_at_deterministic_P(P):
    n, g, r, B, A, lam = 4096, 16, 2, 32, 512, 10
    tau = cm.depth_tau(n, g, r, B)
    mean, se = montecarlo.simulate_mandelbrot_work(n, g, r, tau, P, A, lam, trials=3, seed=W.SEED)
    assert se == 0.0
    assert math.isclose(mean, cm.ssd_work(cm.ModelParams(n, g, r, B, P, A, lam)), rel_tol=1e-12)


@pytest.mark.parametrize("params", [(4096, 16, 2, 32, 0.5, 512, 10), (1024, 4, 4, 4, 0.7, 64, 1),
                                    (2048, 2, 2, 8, 0.75, 2048, 100)])
def test_montecarlo_matches_closed_form(params):
    """Bernoulli-tree mean within 1% (and 4 standard errors)."""
    n, g, r, B, P, A, lam = params
    tau = cm.depth_tau(n, g, r, B)
    mean, se = montecarlo.simulate_mandelbrot_work(n, g, r, tau, P, A, lam, trials=4000, seed=W.SEED)
    w = cm.ssd_work(cm.ModelParams(n, g, r, B, P, A, lam))
    assert abs(mean - w) <= max(4 * se, 1e-9 * w)
    assert abs(mean - w) / w < 0.01


def test_montecarlo_general_form():
    n, g, r, tau = 64, 2, 2, 3
    probs = [0.5, 0.25]
    mean, se = montecarlo.simulate_work(n, g, r, tau, probs, Q=lambda i: 10.0, S=2.0,
                                        T=lambda i: 16.0, A=4.0, trials=20000, seed=W.SEED)
    w = cm.general_subdivision_work(n, g, r, tau, probs, 10.0, 2.0, 16.0, 4.0)
    assert abs(mean - w) <= 4 * se


def test_time_spec_examples():
    # tau=1: T_SBR = A ceil(n^2/(G c)) ceil(G/q) = 512*64*2; T_MBR = A ceil(n^2/(qc))
    p = cm.ModelParams(1024, 16, 2, 64, P=0.5, A=512, lam=10, q=128, c=64)
    assert cm.depth_tau(1024, 16, 2, 64) == 1
    assert cm.sbr_time(p) == 65536
    assert cm.mbr_time(p) == 65536
    assert cm.speedups(p) == (1.0, 1.0)


def _independent_sbr(n, g, r, B, P, A, lam, q, c):
    """Term-by-term exact (Fraction) evaluation of P:300 (SPEC.md S:111 DERIVED check)."""
    from fractions import Fraction as F
    tau = max(1, int(math.floor(math.log(n / (g * B)) / math.log(r) + 1e-9)))
    G, R = g * g, r * r
    Pf, lf = F(P).limit_denominator(1000), F(lam)
    t = F(0)
    for i in range(tau - 1):
        t += (math.ceil(F(4 * n, g * r ** i * c)) * A + Pf * lf * A
              + (1 - Pf) * math.ceil(F(n * n, G * R ** i * c))) * math.ceil(F(G * R ** i, q)) * Pf ** i
    t += A * math.ceil(F(n * n, G * R ** (tau - 1) * c)) * math.ceil(F(G * R ** (tau - 1), q)) * Pf ** (tau - 1)
    return float(t)


def test_sbr_time_exact_summation():
    for args in [(4096, 16, 2, 32, 0.5, 512, 10, 128, 64), (65536, 32, 4, 16, 0.75, 512, 1, 148, 128),
                 (8192, 2, 8, 16, 0.25, 2048, 100, 128, 64)]:
        p = cm.ModelParams(*args)
        assert math.isclose(cm.sbr_time(p), _independent_sbr(*args), rel_tol=1e-12)


def test_bounds_omega_and_speedup():
    """Omega <= A and S <= A over a random parameter sample."""
    rng = np.random.default_rng(W.SEED)
    for _ in range(400):
        n = int(2 ** rng.integers(6, 17))
        g = int(2 ** rng.integers(1, 6))
        B = int(2 ** rng.integers(1, 8))
        if g * B > n:
            continue
        p = cm.ModelParams(n, g, int(2 ** rng.integers(1, 4)), B, float(rng.uniform(0, 1)),
                           float(rng.choice([1, 64, 512, 4096])), float(rng.choice([0, 1, 10, 100])),
                           int(rng.choice([128, 148])), int(rng.choice([64, 128])))
        for mode in ("literal", "leaf"):
            assert cm.work_reduction_factor(p, mode) <= p.A * (1 + 1e-12)
            s1, s2 = cm.speedups(p, mode)
            assert s1 <= p.A * (1 + 1e-12) and s2 <= p.A * (1 + 1e-12)


def test_paper_qualitative_optima():
    """at n=2^16, q=128, c=64, lam <= 100 the optimum speeds up (S > 1) with r ~ 2."""
    for lam in (1, 10, 100):
        (g, r, B), v, _ = cm.grid_search("sbr", 2 ** 16, 0.5, 512, lam)
        te = cm.exhaustive_time(2 ** 16, 128, 64, 512)
        assert te / v > 1 and r == 2
    # minimum work near B ~ 2^3, r ~ 2 ("less work is done near B ~ 2^3")
    (g, r, B), _, _ = cm.grid_search("work", 2 ** 16, 0.5, 512, 10)
    assert r == 2 and 4 <= B <= 16


def test_fit_dimension_recovers_growth():
    regions = [256, 256 * 3, 256 * 9, 256 * 27, 256 * 81]
    D = cm.fit_dimension(regions, 2)
    assert abs(D - math.log2(3)) < 1e-9
    assert abs(2 ** (D - 2) - 0.75) < 1e-9


def test_fit_lambda_roundtrip():
    p = cm.ModelParams(8192, 16, 2, 32, 0.75, 2048, 37.0, 148, 128)
    t_unit = 1e-9
    t = cm.sbr_time(p, "leaf") * t_unit
    lam = cm.fit_lambda(t, t_unit, p, "leaf")
    assert abs(lam - 37.0) < 1e-6


def test_spearman():
    assert cm.spearman([1, 2, 3], [10, 20, 30]) == 1.0
    assert cm.spearman([1, 2, 3], [3, 2, 1]) == -1.0


def test_mbr_time_special_cases():
    """T_MBR at its two degenerate subdivision probabilities.  P = 0: every level-0
    region is uniform, so one parallel border pass over the g^2 regions plus one flat fill of
    the n^2 pixels.  P = 1: every region subdivides, so no fill at all and the last level
    computes every pixel (A ceil(n^2/(qc))), plus per level the border pass and the
    subdivision cost S = lam A per region."""
    n, g, r, B, A, lam, q, c = 8192, 16, 2, 32, 512.0, 3.0, 148, 128
    tau = cm.depth_tau(n, g, r, B)
    assert tau >= 2
    G = g * g
    p0 = cm.ModelParams(n, g, r, B, 0.0, A, lam, q, c)
    assert cm.mbr_time(p0) == math.ceil(4 * n / (g * c)) * math.ceil(G / q) * A + math.ceil(n * n / (q * c))
    p1 = cm.ModelParams(n, g, r, B, 1.0, A, lam, q, c)
    want = A * math.ceil(n * n / (q * c))
    for i in range(tau - 1):
        Gi = G * (r * r) ** i
        want += math.ceil(4 * n / (g * r ** i * c)) * math.ceil(Gi / q) * A + math.ceil(Gi / q) * lam * A
    assert math.isclose(cm.mbr_time(p1), want, rel_tol=1e-12)


def test_fit_lambda_roundtrip_mbr():
    """The per-scheme calibration (sweep_c2 fits lambda with the scheme's own model)."""
    p = cm.ModelParams(8192, 16, 2, 32, 0.6, 2048, 11.0, 148, 128)
    t_unit = 2e-9
    t = cm.mbr_time(p, "leaf") * t_unit
    assert abs(cm.fit_lambda(t, t_unit, p, "leaf", scheme="mbr") - 11.0) < 1e-6
    cal = cm.calibrate(8192, 2048.0, cm.exhaustive_time(8192, 148, 128, 2048.0) * t_unit, (16, 2, 32),
                       [256, 256 * 3, 256 * 9, 256 * 27], t, scheme="mbr")
    assert cal.scheme == "mbr" and abs(cal.t_unit - t_unit) < 1e-18


def test_landscapes_tool_runs():
    """tools/landscapes.py (NEXT-2) evaluates the figure data; Omega stays below A and the
    claims report is complete."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "landscapes", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "landscapes.py"))
    L = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(L)
    e1 = L.e1()
    for A, ws in e1["omega_n_vs_A"].items():
        assert all(w <= A * (1 + 1e-12) for w in ws)
    e2 = L.e2(cm.B200_Q, cm.B200_C)
    assert set(e2["S_param"]) == {"g", "r", "B"}
    cl = L.claims(e1, e2)
    assert cl["Omega <= A everywhere (P:244)"] and len(cl) >= 10
