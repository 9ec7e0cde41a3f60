"""Pins for multi-step decision periods (PAPER.md:78-79,
:130 "the period between forecasts and power limit adjustments"; SPEC.md:158-166
forecast_horizon, :348 mean-of-horizon decision).

At each period start w the forecaster runs recursively from the last observed
value over n = min(P, N - w) steps (prediction k is the lag of prediction
k+1, clamped at 0), Eq. 6 takes the mean of those n forecasts, and every
window of the period gets that decision.
"""
import json
import os
from fractions import Fraction as F

import numpy as np

import oracle
from oracle import exact
from conftest import GOLDEN

# exact phase features for T = 4: (sin, cos) at phi = 0, 1, 2, 3
SC4 = {0: (0, 1), 1: (1, 0), 2: (0, -1), 3: (-1, 0)}


def test_horizon_recursion_matches_exact_rationals():
    """T=4 golden model (beta exact, tests/golden/fit_t4.json), period 3 from
    w = 6: the hand-unrolled recursion in exact rationals (S:166 DERIVED)."""
    g = json.load(open(os.path.join(GOLDEN, "fit_t4.json")))
    hist = [float(v) for v in g["history"]]          # 6 points, T = 4
    beta = [F(b) for b in g["beta_intercept_sin_cos_lag"]]
    future = [480.0, 430.0, 470.0, 520.0, 505.0]     # windows 6..10: periods [6,9) and [9,11)
    c = np.array(hist + future)
    L, T, P = len(hist), 4, 3
    prof = dict(avg_power=[150.0, 240.0, 290.0], thr=[500.0, 700.0, 800.0])
    fc, ch, tot, st = oracle.plan_trace(c, L=L, T=T, period=P, etas=[0.5], pmax=300.0, max_ci=750.0, **prof)
    assert st == 0

    def horizon(w, n):
        prev, out = F(c[w - 1]), []
        for k in range(n):
            s, co = SC4[(w + k) % 4]
            f = beta[0] + beta[1] * s + beta[2] * co + beta[3] * prev
            f = max(f, F(0))
            out.append(f)
            prev = f
        return sum(out) / n

    for w0, n in [(6, 3), (9, 2)]:
        m = horizon(w0, n)
        for k in range(n):
            assert abs(fc[w0 - L + k] - float(m)) <= 1e-12 * float(m)
        # the decision is the exact Eq. 6 argmin at the exact mean (clear of ties here)
        costs = exact.costs(F(1, 2), prof["avg_power"], prof["thr"], F(300), F(750), m)
        k_star = exact.argmin_first(costs)
        assert exact.rel_gap_top2(costs) > 1e-9
        assert list(ch[0, w0 - L:w0 - L + n]) == [k_star] * n


def test_period_one_is_the_per_window_planner():
    rng = np.random.default_rng(5)
    T, L, N = 24, 24, 24 + 200
    c = np.round((500 + 120 * np.sin(2 * np.pi * np.arange(N) / T) + rng.normal(0, 20, N)) * 64) / 64
    kw = dict(L=L, T=T, avg_power=[100.0, 200.0, 280.0], thr=[400.0, 700.0, 780.0], etas=[0.3, 0.7], pmax=300.0,
              J=3600 * 150 * 400.0)
    a = oracle.plan_trace(c, **kw)
    b = oracle.plan_trace(c, period=1, **kw)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    # and the per-window decision is Eq. 6 on the one-step forecast with the observed lag
    m = oracle.fit(c[:L], T=T)
    S, C = oracle.phase_table(T)
    for w in (L, L + 7, N - 1):
        chat = oracle.predict(m, S[w % T], C[w % T], c[w - 1])
        assert a[0][w - L] == chat


def test_decisions_constant_within_periods_and_partial_last_period():
    rng = np.random.default_rng(9)
    T, L, N, P = 24, 24, 24 + 100, 7                     # W = 100: 14 periods of 7, then one of 2
    c = np.round((450 + 150 * np.sin(2 * np.pi * np.arange(N) / T) + rng.normal(0, 25, N)) * 64) / 64
    fc, ch, tot, st = oracle.plan_trace(c, L=L, T=T, period=P, avg_power=[100.0, 200.0, 280.0],
                                        thr=[400.0, 700.0, 780.0], etas=[0.5, 0.9], pmax=300.0)
    assert st == 0
    for start in range(0, 100, P):
        seg = slice(start, min(start + P, 100))
        assert len(set(fc[seg])) == 1
        for e in range(2):
            assert len(set(ch[e, seg])) == 1
    # the last, partial period averages only its 2 windows: recompute its horizon
    m = oracle.fit(c[:L], T=T)
    S, C = oracle.phase_table(T)
    w0 = L + 98
    f1 = oracle.predict(m, S[w0 % T], C[w0 % T], c[w0 - 1])
    f2 = oracle.predict(m, S[(w0 + 1) % T], C[(w0 + 1) % T], f1)
    assert fc[98] == (0.0 + f1 + f2) / 2.0


def test_constant_history_gives_constant_decisions():
    T, L, N = 24, 24, 24 + 60
    c = np.full(N, 321.0)
    fc, ch, tot, st = oracle.plan_trace(c, L=L, T=T, period=12, avg_power=[100.0, 200.0], thr=[400.0, 700.0],
                                        etas=[0.5], pmax=300.0)
    assert st == 0 and np.all(fc == 321.0) and len(set(ch[0])) == 1
