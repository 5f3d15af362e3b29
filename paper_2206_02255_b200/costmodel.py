"""The paper's subdivision cost model (Sec. 4), host-side, plus the calibration
and {g, r, B} predictor of SURVEY.md §8(c) c-6 (row a12 of the hot-path table).

Pure Python/float64 closed forms, evaluated literally as printed (R10-R12):
  W_E            = n^2 A                                    P:112-117 eq:exhaustive-general
  W_S (general)  = sum_{i=0}^{tau-2} U_i G R^i prod_{j<i} P_j + n^2 A prod_{j<=tau-2} P_j
                   U_i = P_i (Q+S) + (1-P_i)(Q+T)           P:176-181 eq:...-general-expanded
  W^M_SSD        = sum_{i=0}^{tau-2} [4nA/(g r^i) + P lam A + (1-P) n^2/(G R^i)] G R^i P^i
                   + n^2 A P^(tau-1)
  Omega          = W_E / W^M_SSD
  T_Ex           = ceil(n^2/(qc)) A                          P:283-286 eq:time-exhaustive
  T_SBR, T_MBR   = the two eq:time-subdiv-QT
  S_SBR, S_MBR   = T_Ex / T_SBR, T_Ex / T_MBR
with G = g^2, R = r^2, S = lam A and tau = log_r(n/(gB)).

tau convention (R5): the paper's literal tau = floor(log_r(n/(gB))) (clamped to
>= 1) makes the last-level side rB; the built ASK stops when d/r < B, i.e. it runs
tau + 1 levels with leaf side B.  Every function takes `tau_mode` = "literal" | "leaf".
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

B200_Q = 148   # SMs
B200_C = 128   # FP32 lanes per SM
PAPER_Q, PAPER_C = 128, 64


@dataclasses.dataclass(frozen=True)
class ModelParams:
    """All cost-model symbols (SPEC.md S:27-33 ModelParams)."""
    n: int
    g: int
    r: int
    B: int
    P: float = 0.5
    A: float = 512.0
    lam: float = 1.0
    q: int = PAPER_Q
    c: int = PAPER_C

    def validate(self) -> None:
        for name in ("n", "g", "r", "B"):
            v = getattr(self, name)
            if v < 1 or v & (v - 1):
                raise ValueError(f"{name}={v} must be a power of two")
        if self.r < 2:
            raise ValueError("r must be >= 2")
        if self.g * self.B > self.n:
            raise ValueError("g*B must be <= n")
        if not 0.0 <= self.P <= 1.0:
            raise ValueError("P must be in [0, 1]")
        if self.A < 1 or self.lam < 0 or self.q < 1 or self.c < 1:
            raise ValueError("A >= 1, lam >= 0, q >= 1, c >= 1")


def _ilog(x: int, base: int) -> int:
    """floor(log_base(x)) for integers x >= 1, exactly."""
    k = 0
    while x >= base:
        x //= base
        k += 1
    return k


def depth_tau(n: int, g: int, r: int, B: int, tau_mode: str = "literal") -> int:
    """tau = log_r(n/(gB)), floored and clamped to >= 1.  "leaf" adds one level,
    which is the number of levels the built ASK runs (leaf side B)."""
    if g * B > n:
        raise ValueError("g*B > n: no valid depth")
    t = _ilog(n // (g * B), r)
    if tau_mode == "literal":
        return max(1, t)
    if tau_mode == "leaf":
        return t + 1
    raise ValueError(tau_mode)


def exhaustive_work(n: int, A: float) -> float:
    """W_E = n^2 A."""
    return float(n) * n * A


def general_subdivision_work(n: int, g: int, r: int, tau: int, probs: Sequence[float],
                             Q: float, S: float, T: float, A: float) -> float:
    """W_S(n) with per-level P_0..P_{tau-2} and per-region constants Q, S, T."""
    if len(probs) != max(0, tau - 1):
        raise ValueError("need tau-1 probabilities")
    G, R = g * g, r * r
    K = 0.0
    prod = 1.0
    for i in range(tau - 1):
        U = probs[i] * (Q + S) + (1.0 - probs[i]) * (Q + T)
        K += U * G * R ** i * prod
        prod *= probs[i]
    return K + float(n) * n * A * prod


def ssd_work_terms(p: ModelParams, tau: int) -> Tuple[List[float], float]:
    """Per-level K_i and L of W^M_SSD (Mandelbrot instantiation)."""
    n, g, r, P, A, lam = p.n, p.g, p.r, p.P, p.A, p.lam
    G, R = g * g, r * r
    K = []
    for i in range(tau - 1):
        Qi = 4.0 * n * A / (g * r ** i)
        Ti = float(n) * n / (G * R ** i)
        K.append((Qi + P * lam * A + (1.0 - P) * Ti) * G * R ** i * P ** i)
    L = float(n) * n * A * P ** (tau - 1)
    return K, L


def ssd_work(p: ModelParams, tau_mode: str = "literal") -> float:
    """W^M_SSD."""
    K, L = ssd_work_terms(p, depth_tau(p.n, p.g, p.r, p.B, tau_mode))
    return sum(K) + L


def work_reduction_factor(p: ModelParams, tau_mode: str = "literal") -> float:
    """Omega = W_E / W^M_SSD."""
    return exhaustive_work(p.n, p.A) / ssd_work(p, tau_mode)


def _ceil(x: float) -> float:
    return float(math.ceil(x - 1e-12 * abs(x)))


def exhaustive_time(n: int, q: int, c: int, A: float) -> float:
    """T_Ex = ceil(n^2/(qc)) A."""
    return float(-(-(n * n) // (q * c))) * A


def sbr_time(p: ModelParams, tau_mode: str = "literal") -> float:
    """T_SBR, the first eq:time-subdiv-QT, literally (R11):
    sum_{i=0}^{tau-2} (ceil(4n/(g r^i c)) A + P lam A + (1-P) ceil(n^2/(G R^i c)))
                      * ceil(G R^i / q) * P^i
    + A ceil(n^2/(G R^(tau-1) c)) ceil(G R^(tau-1)/q) P^(tau-1)."""
    n, g, r, P, A, lam, q, c = p.n, p.g, p.r, p.P, p.A, p.lam, p.q, p.c
    tau = depth_tau(n, g, r, p.B, tau_mode)
    G, R = g * g, r * r
    t = 0.0
    for i in range(tau - 1):
        Gi = G * R ** i
        term = (-(-(4 * n) // (g * r ** i * c))) * A + P * lam * A \
            + (1.0 - P) * (-(-(n * n) // (Gi * c)))
        t += term * (-(-Gi // q)) * P ** i
    Gl = G * R ** (tau - 1)
    t += A * (-(-(n * n) // (Gl * c))) * (-(-Gl // q)) * P ** (tau - 1)
    return t


def mbr_time(p: ModelParams, tau_mode: str = "literal") -> float:
    """T_MBR, the second eq:time-subdiv-QT, literally:
    sum_{i=0}^{tau-2} ( ceil(4n/(g r^i c)) ceil(G R^i/q) A P^i + ceil(G R^i/q) S P^(i+1)
                        + ceil(n^2 P^i (1-P)/(qc)) ) + A ceil(n^2/(qc)) P^(tau-1)."""
    n, g, r, P, A, lam, q, c = p.n, p.g, p.r, p.P, p.A, p.lam, p.q, p.c
    tau = depth_tau(n, g, r, p.B, tau_mode)
    G, R = g * g, r * r
    S = lam * A
    t = 0.0
    for i in range(tau - 1):
        Gi = G * R ** i
        t += (-(-(4 * n) // (g * r ** i * c))) * (-(-Gi // q)) * A * P ** i
        t += (-(-Gi // q)) * S * P ** (i + 1)
        t += _ceil(float(n) * n * P ** i * (1.0 - P) / (q * c))
    t += A * (-(-(n * n) // (q * c))) * P ** (tau - 1)
    return t


def speedups(p: ModelParams, tau_mode: str = "literal") -> Tuple[float, float]:
    """(S_SBR, S_MBR) = T_Ex / T_scheme."""
    te = exhaustive_time(p.n, p.q, p.c, p.A)
    return te / sbr_time(p, tau_mode), te / mbr_time(p, tau_mode)


# --------------------------------------------------------------------------- search
POW2_SPACE = tuple(2 ** k for k in range(1, 11))  # {2..1024}


def grid_search(objective: str, n: int, P: float, A: float, lam: float,
                q: int = PAPER_Q, c: int = PAPER_C, g_set=POW2_SPACE, r_set=POW2_SPACE,
                B_set=POW2_SPACE, tau_mode: str = "literal",
                P_of_r=None) -> Tuple[Tuple[int, int, int], float, Dict]:
    """argmin over feasible {g, r, B} of "work" (W^M_SSD), "sbr" or "mbr" time (P:242,
    P:320).  Ties break to the lexicographically smallest (g, r, B).  P_of_r, if given,
    maps r -> P (the SSD law P = r^(D-2), R12)."""
    best, best_v, land = None, math.inf, {}
    for g in g_set:
        for r in r_set:
            for B in B_set:
                if g * B > n:
                    continue
                pp = ModelParams(n, g, r, B, P if P_of_r is None else P_of_r(r), A, lam, q, c)
                if objective == "work":
                    v = ssd_work(pp, tau_mode)
                elif objective == "sbr":
                    v = sbr_time(pp, tau_mode)
                elif objective == "mbr":
                    v = mbr_time(pp, tau_mode)
                else:
                    raise ValueError(objective)
                land[(g, r, B)] = v
                if v < best_v:
                    best, best_v = (g, r, B), v
    return best, best_v, land


# --------------------------------------------------------------------------- calibration
def fit_dimension(level_regions: Sequence[int], r: int) -> float:
    """Box-counting dimension D from regions_l ~ (r^D)^l (least squares on
    log regions_l vs l log r over l >= 1).  Then P(r) = r^(D-2)."""
    pts = [(l, math.log(v)) for l, v in enumerate(level_regions) if l >= 1 and v > 0]
    if len(pts) < 2:
        pts = [(l, math.log(v)) for l, v in enumerate(level_regions) if v > 0]
    if len(pts) < 2:
        return 2.0
    xs = [l * math.log(r) for l, _ in pts]
    ys = [y for _, y in pts]
    mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
    sxx = sum((x - mx) ** 2 for x in xs)
    sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    return sxy / sxx


def scheme_time(p: ModelParams, scheme: str = "sbr", tau_mode: str = "literal") -> float:
    """T_SBR or T_MBR by name."""
    if scheme == "sbr":
        return sbr_time(p, tau_mode)
    if scheme == "mbr":
        return mbr_time(p, tau_mode)
    raise ValueError(scheme)


def fit_lambda(t_ask: float, t_unit: float, p: ModelParams, tau_mode: str = "leaf",
               scheme: str = "sbr") -> float:
    """Solve T_scheme(lam) * t_unit = t_ask for lam.  T_SBR and T_MBR are affine in lam."""
    p0 = dataclasses.replace(p, lam=0.0)
    p1 = dataclasses.replace(p, lam=1.0)
    a0, a1 = scheme_time(p0, scheme, tau_mode), scheme_time(p1, scheme, tau_mode)
    slope = a1 - a0
    if slope <= 0:
        return 0.0
    return max(0.0, (t_ask / t_unit - a0) / slope)


@dataclasses.dataclass
class Calibration:
    t_unit: float      # seconds per model time unit (from the exhaustive run)
    D: float           # fitted box-counting dimension
    lam: float         # fitted subdivision cost multiplier
    A: float
    q: int
    c: int
    tau_mode: str
    scheme: str = "sbr"

    def P(self, r: int) -> float:
        return min(1.0, max(0.0, r ** (self.D - 2.0)))

    def predict_time(self, n: int, g: int, r: int, B: int) -> float:
        p = ModelParams(n, g, r, B, self.P(r), self.A, self.lam, self.q, self.c)
        return scheme_time(p, self.scheme, self.tau_mode) * self.t_unit


def calibrate(n: int, A: float, t_ex: float, ref: Tuple[int, int, int], ref_level_regions:
              Sequence[int], t_ref: float, q: int = B200_Q, c: int = B200_C,
              tau_mode: str = "leaf", scheme: str = "sbr") -> Calibration:
    """SURVEY.md c-6 protocol: t_unit from the exhaustive run alone, D (hence P) from the
    reference run's level sizes, lam from the reference run's time (T_SBR or T_MBR)."""
    t_unit = t_ex / exhaustive_time(n, q, c, A)
    g, r, B = ref
    D = fit_dimension(ref_level_regions, r)
    P = min(1.0, max(0.0, r ** (D - 2.0)))
    lam = fit_lambda(t_ref, t_unit, ModelParams(n, g, r, B, P, A, 0.0, q, c), tau_mode, scheme)
    return Calibration(t_unit, D, lam, A, q, c, tau_mode, scheme)


def spearman(a: Sequence[float], b: Sequence[float]) -> float:
    def ranks(v):
        order = sorted(range(len(v)), key=lambda i: v[i])
        rk = [0.0] * len(v)
        i = 0
        while i < len(order):
            j = i
            while j + 1 < len(order) and v[order[j + 1]] == v[order[i]]:
                j += 1
            for k in range(i, j + 1):
                rk[order[k]] = (i + j) / 2.0
            i = j + 1
        return rk
    ra, rb = ranks(list(a)), ranks(list(b))
    n = len(a)
    ma, mb = sum(ra) / n, sum(rb) / n
    num = sum((x - ma) * (y - mb) for x, y in zip(ra, rb))
    den = math.sqrt(sum((x - ma) ** 2 for x in ra) * sum((y - mb) ** 2 for y in rb))
    return num / den if den else 0.0
