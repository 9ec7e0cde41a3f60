"""Exact-rational micro-oracle (TEST INFRASTRUCTURE).

Independent of liboracle: computes the same quantities in exact rational
arithmetic (fractions.Fraction), so the fp64 oracle can be pinned to the
mathematics rather than to itself:
  - least squares with intercept via exact normal equations (Eq. 1),
  - the exact Eq. 6 cost vector and its argmin,
  - the fixed-work stepwise replay.
"""
from __future__ import annotations

from fractions import Fraction as F


def _solve(A, b):
    """Gauss-Jordan elimination over Fractions (A square, nonsingular)."""
    n = len(A)
    M = [list(map(F, row)) + [F(b[i])] for i, row in enumerate(A)]
    for col in range(n):
        piv = next(r for r in range(col, n) if M[r][col] != 0)
        M[col], M[piv] = M[piv], M[col]
        pv = M[col][col]
        M[col] = [v / pv for v in M[col]]
        for r in range(n):
            if r != col and M[r][col] != 0:
                fct = M[r][col]
                M[r] = [a - fct * c for a, c in zip(M[r], M[col])]
    return [M[i][n] for i in range(n)]


def lstsq_intercept(X, y):
    """Exact OLS of y on [1, X]: returns [b0, b1, ..., bp] as Fractions."""
    rows = [[F(1)] + [F(v) for v in r] for r in X]
    p = len(rows[0])
    A = [[sum(r[i] * r[j] for r in rows) for j in range(p)] for i in range(p)]
    b = [sum(r[i] * F(yy) for r, yy in zip(rows, y)) for i in range(p)]
    return _solve(A, b)


def costs(eta, avg_power, thr, pmax, maxci, chat):
    """Exact Eq. 6 numerator/Throughput (no 3.6e6 divisor, DESIGN Q12)."""
    eta, pmax, maxci, chat = F(eta), F(pmax), F(maxci), F(chat)
    return [(eta * F(p) * chat + (1 - eta) * pmax * maxci) / F(t) for p, t in zip(avg_power, thr)]


def argmin_first(vals):
    best = 0
    for k in range(1, len(vals)):
        if vals[k] < vals[best]:
            best = k
    return best


def rel_gap_top2(vals):
    s = sorted(vals)
    if s[0] == 0:
        return F(0) if s[1] == 0 else F(10**9)
    return (s[1] - s[0]) / s[0]


def replay(c, s0, choice, avg_power, thr, delta, J):
    """Exact stepwise fixed-work replay; returns (time, energy, carbon, samples, w*, status)."""
    S = E = C = F(0)
    delta, J = F(delta), F(J)
    for w in range(s0, len(c)):
        k = choice[w - s0]
        sk = F(thr[k]) * delta
        prev = S
        S = S + sk
        if J > 0 and S >= J:
            f = (J - prev) / sk
            return ((w - s0 + f) * delta, (E + f * F(avg_power[k])) * delta,
                    (C + f * F(avg_power[k]) * F(c[w])) * delta / F(3600000), J, w, 0)
        E += F(avg_power[k])
        C += F(avg_power[k]) * F(c[w])
    return ((len(c) - s0) * delta, E * delta, C * delta / F(3600000), S, -1, 3 if J > 0 else 0)
