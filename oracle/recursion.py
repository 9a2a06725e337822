"""Idealised branching-process recursions (TEST INFRASTRUCTURE ONLY).

Double precision, written in the paper's notation.  Used only to pin the
oracle's peel against the paper's printed predictions and laws:

* ``plain(c, r, k, T)``      -- rho_i, lambda_i, beta_i of P:121-144
* ``c_star(r, k)``           -- threshold; for k=2 the closed form of P:96
* ``contraction(c, r, k)``   -- fixed point beta and factor a of P:329-341
* ``subtable(c, r, k, I)``   -- rho_{i,j}, lambda_{i,j}, lambda'_{i,j} of P:583-597
* ``round_bound(n, r, k)``   -- log log n / log((k-1)(r-1)) of P:16
"""
from __future__ import annotations

import math

from scipy.optimize import minimize_scalar


def poisson_tail(beta: float, j: int) -> float:
    """Pr(Poisson(beta) >= j) = 1 - e^{-beta} sum_{i<j} beta^i / i!.

    For beta < j the same quantity is summed as the upper tail
    e^{-beta} sum_{i>=j} beta^i / i! so that tiny values (lambda_t down to
    1e-300 below threshold) do not cancel to zero."""
    if j <= 0:
        return 1.0
    if beta < j:
        term = math.exp(-beta)
        for i in range(1, j + 1):
            term *= beta / i
        s, i = 0.0, j
        while term > 0.0 and term > 1e-18 * s:
            s += term
            i += 1
            term *= beta / i
        return s
    s, term = 0.0, 1.0
    for i in range(j):
        if i > 0:
            term *= beta / i
        s += term
    return 1.0 - math.exp(-beta) * s


def plain(c: float, r: int, k: int, T: int):
    """rho_0 = 1; beta_i = rho_{i-1}^{r-1} r c;
    rho_i = Pr(Po(beta_i) >= k-1); lambda_i = Pr(Po(beta_i) >= k).

    Returns lists (beta[1..T], rho[0..T], lam[1..T]) as 0-based python lists
    with beta[0] = beta_1, rho[0] = rho_0, lam[0] = lambda_1.
    """
    rho = [1.0]
    beta, lam = [], []
    for i in range(1, T + 1):
        b = rho[i - 1] ** (r - 1) * r * c
        beta.append(b)
        rho.append(poisson_tail(b, k - 1))
        lam.append(poisson_tail(b, k))
    return beta, rho, lam


def c_star(r: int, k: int) -> float:
    """Threshold c*_{k,r} = min_{x>0} x / (r Pr[Po(x) >= k-1]^{r-1}).

    For k = 2 this is the paper's closed form min_x x / (r (1-e^{-x})^{r-1})
    (P:96); for general k the same minimisation with the Poisson tail (the
    fixed-point condition of the beta map)."""
    f = lambda x: x / (r * poisson_tail(x, k - 1) ** (r - 1))
    res = minimize_scalar(f, bounds=(1e-6, 50.0), method="bounded",
                          options={"xatol": 1e-12})
    return float(res.fun)


def contraction(c: float, r: int, k: int, iters: int = 200000):
    """Above threshold: fixed point beta of P:331 by iteration from beta_1 = rc,
    and a = (r-1) beta e^{-beta} S_{k-2} (1 - S_{k-3}/S_{k-2}) / (1 - e^{-beta} S_{k-2})
    (P:341), with S_j = sum_{h<=j} beta^h/h! and S_{k-3} = 0 for k = 2.
    Returns (beta, a, lambda) with lambda = 1 - e^{-beta} S_{k-1}."""
    beta = r * c
    for _ in range(iters):
        nb = poisson_tail(beta, k - 1) ** (r - 1) * r * c
        if abs(nb - beta) < 1e-15:
            beta = nb
            break
        beta = nb

    def S(j):
        if j < 0:
            return 0.0
        return sum(beta ** h / math.factorial(h) for h in range(j + 1))

    Sk2, Sk3 = S(k - 2), S(k - 3)
    a = (r - 1) * beta * math.exp(-beta) * Sk2 * (1 - Sk3 / Sk2) / (1 - math.exp(-beta) * Sk2)
    lam = 1 - math.exp(-beta) * S(k - 1)
    return beta, a, lam


def subtable(c: float, r: int, k: int, I: int):
    """Subtable recursion and lambda'.

    rho_{0,j} = 1, lambda_{0,j} = 1;
    beta_{i,j} = prod_{h<j} rho_{i,h} prod_{h>j} rho_{i-1,h} r c;
    rho_{i,j} = Pr(Po(beta_{i,j}) >= k-1); lambda_{i,j} = Pr(Po(beta_{i,j}) >= k);
    lambda'_{i,j} = (1/r)(sum_{h<=j} lambda_{i,h} + sum_{h>j} lambda_{i-1,h}).
    Returns lam_prime as a list of (i, j, value) for i=1..I, j=1..r.
    """
    rho_prev = [1.0] * r
    lam_prev = [1.0] * r
    out = []
    for i in range(1, I + 1):
        rho_cur = [0.0] * r
        lam_cur = [0.0] * r
        for j in range(r):
            b = r * c
            for h in range(j):
                b *= rho_cur[h]
            for h in range(j + 1, r):
                b *= rho_prev[h]
            rho_cur[j] = poisson_tail(b, k - 1)
            lam_cur[j] = poisson_tail(b, k)
            lp = (sum(lam_cur[: j + 1]) + sum(lam_prev[j + 1:])) / r
            out.append((i, j + 1, lp))
        rho_prev, lam_prev = rho_cur, lam_cur
    return out


def round_bound(n: float, r: int, k: int) -> float:
    """t* leading term log log n / log((k-1)(r-1))."""
    return math.log(math.log(n)) / math.log((k - 1) * (r - 1))
