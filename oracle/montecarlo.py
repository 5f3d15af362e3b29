"""Monte-Carlo subdivision-tree oracle for the cost model — TEST INFRASTRUCTURE ONLY.

Simulates the random process the cost model's expectation describes (Sec. 4.2):
starting from G = g^2 regions, at each level i = 0..tau-2 every region independently
subdivides with probability P_i, paying Q_i + S, or terminates, paying Q_i + T_i; a
subdividing region creates R = r^2 regions at level i+1.  Regions that reach level tau-1
pay the last-level work (n^2 / (G R^(tau-1))) * A each.  The mean total work
over trials estimates W_S; the closed forms in costmodel must match it.

Plain numpy; the level-by-level count process draws Binomial(count, P_i) subdividers,
which is the same distribution as per-region Bernoulli draws.
"""
from __future__ import annotations

from typing import Callable, Sequence, Tuple

import numpy as np


def simulate_work(n: int, g: int, r: int, tau: int, probs: Sequence[float],
                  Q: Callable[[int], float], S: float, T: Callable[[int], float], A: float,
                  trials: int, seed: int) -> Tuple[float, float]:
    """Returns (mean total work, standard error of the mean)."""
    rng = np.random.default_rng(seed)
    G, R = g * g, r * r
    totals = np.zeros(trials)
    for t in range(trials):
        count = G
        work = 0.0
        for i in range(tau - 1):
            sub = int(rng.binomial(count, probs[i]))
            work += sub * (Q(i) + S) + (count - sub) * (Q(i) + T(i))
            count = sub * R
        work += count * (float(n) * n / (G * R ** (tau - 1))) * A
        totals[t] = work
    return float(totals.mean()), float(totals.std(ddof=1) / np.sqrt(trials)) if trials > 1 else 0.0


def simulate_mandelbrot_work(n: int, g: int, r: int, tau: int, P: float, A: float, lam: float,
                             trials: int, seed: int) -> Tuple[float, float]:
    """Mandelbrot instantiation: Q_i = 4nA/(g r^i), T_i = n^2/(G R^i), S = lam A."""
    G, R = g * g, r * r
    return simulate_work(n, g, r, tau, [P] * (tau - 1),
                         Q=lambda i: 4.0 * n * A / (g * r ** i), S=lam * A,
                         T=lambda i: float(n) * n / (G * R ** i), A=A, trials=trials, seed=seed)
