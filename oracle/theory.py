"""Collision probabilities and moments used as statistical pins — TEST INFRASTRUCTURE ONLY.

These are the paper's stated collision behaviour and its exact counterparts; the tests compare the
empirical collision rates of the hashing oracle against them, which pins the oracle's arithmetic
to something other than itself.
"""
from __future__ import annotations

import itertools
import math

import numpy as np


def Phi(x: float) -> float:
    return 0.5 * math.erfc(-x / math.sqrt(2.0))


def p_e2lsh(s: float, w: float) -> float:
    """E2LSH collision probability, Eq. 2 in closed form:
    p(s) = 2 Phi(w/s) - 1 - (2 s / (sqrt(2 pi) w)) (1 - exp(-w^2 / (2 s^2))),  p(0) = 1."""
    if s <= 0.0:
        return 1.0
    r = w / s
    return 2.0 * Phi(r) - 1.0 - (2.0 / (math.sqrt(2.0 * math.pi) * r)) * (1.0 - math.exp(-r * r / 2.0))


def p_e2lsh_integral(s: float, w: float) -> float:
    """Eq. 2 by numerical quadrature of int_0^w f_{|sX|}(t) (1 - t/w) dt, f_{|sX|}(t) = (2/s) phi(t/s).
    Independent of the closed form above (used to pin it)."""
    from scipy.integrate import quad

    def f(t):
        return (2.0 / s) * math.exp(-0.5 * (t / s) ** 2) / math.sqrt(2.0 * math.pi) * (1.0 - t / w)

    val, _ = quad(f, 0.0, w, epsabs=1e-13, epsrel=1e-12, limit=200)
    return val


def p_fastlsh_exact_enum(v, u, m: int, w: float) -> float:
    """Exact FastLSH collision probability for tiny n, m:
    conditional on S, a.(S(v)-S(u)) ~ N(0, ||S(v-u)||^2) by 2-stability, so
    p = E_S[ p_e2lsh(||S(v-u)||; w) ], enumerated over all n^m equally likely index tuples."""
    d2 = [(float(a) - float(b)) ** 2 for a, b in zip(v, u)]
    n = len(d2)
    tot = 0.0
    for S in itertools.product(range(n), repeat=m):
        tot += p_e2lsh(math.sqrt(sum(d2[i] for i in S)), w)
    return tot / n ** m


def p_fastlsh_exact_mc(v, u, m: int, w: float, draws: int = 200_000, seed: int = 0) -> float:
    """Same expectation by Monte Carlo over S with the closed-form inner term (for larger n, m)."""
    d2 = (np.asarray(v, np.float64) - np.asarray(u, np.float64)) ** 2
    rng = np.random.default_rng(seed)
    S = rng.integers(0, d2.shape[0], size=(draws, m))
    s = np.sqrt(d2[S].sum(axis=1))
    r = np.where(s > 0, w / np.maximum(s, 1e-300), np.inf)
    from scipy.special import erf
    phi2 = erf(r / math.sqrt(2.0))  # 2 Phi(r) - 1
    tail = np.where(np.isfinite(r), (2.0 / (math.sqrt(2.0 * math.pi) * r)) * (1.0 - np.exp(-r * r / 2.0)), 0.0)
    return float(np.mean(np.where(s > 0, phi2 - tail, 1.0)))


def pair_stats(v, u):
    """(s, mu, sigma^2) of the population {(v_i - u_i)^2}."""
    d2 = (np.asarray(v, np.float64) - np.asarray(u, np.float64)) ** 2
    return math.sqrt(d2.sum()), float(d2.mean()), float(d2.var())


def exact_moments(v, u, m: int):
    """Exact E[dP^2], E[dP^4] for dP = a.(S(v) - S(u)) (untruncated counterpart of Lemma 4.8,
    PAPER.md:308-323): E[dP^2] = m s^2 / n, E[dP^4] = 3 (m sigma^2 + m^2 mu^2)."""
    s, mu, var = pair_stats(v, u)
    n = len(v)
    return m * s * s / n, 3.0 * (m * var + m * m * mu * mu)


def p_fastlsh_eq9(v, u, m: int, w: float) -> float:
    """The paper's Thm 4.4 / Eq. 9, evaluated as the 1-D mixture
    int_0^inf psi(y; mu~, sigma~^2, 0, inf) p_e2lsh(sqrt(y); w) dy with mu~ = m mu,
    sigma~^2 = m sigma^2 (Eqs. 6-7). A CLT approximation of the exact value."""
    from scipy.integrate import quad
    _, mu, var = pair_stats(v, u)
    mt, st = m * mu, math.sqrt(m * var)
    Z = 1.0 - Phi(-mt / st)

    def f(y):
        return math.exp(-0.5 * ((y - mt) / st) ** 2) / (st * math.sqrt(2 * math.pi)) / Z * p_e2lsh(math.sqrt(y), w)

    lo, hi = max(0.0, mt - 12 * st), mt + 12 * st
    val, _ = quad(f, lo, hi, limit=400, epsabs=1e-12, epsrel=1e-10)
    return val


def width_equivalent(w: float, m: int, n: int) -> float:
    """w~ = sqrt(m/n) w — the width at which FastLSH matches E2LSH asymptotically
    (Cor. 4.7, read with Fact 4.5 — DESIGN.md reading R7)."""
    return math.sqrt(m / n) * w
