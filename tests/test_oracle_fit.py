"""Pins for the oracle's Eq. 1-2 forecaster.

Each test ties oracle_fit / oracle_predict to something other than itself:
closed-form features, exact rational least squares, numpy's SVD lstsq (a
different algorithm), and the SPEC special cases.
"""
import json
import math
import os
from fractions import Fraction as F

import numpy as np
import pytest

import oracle
from oracle import exact
from conftest import GOLDEN


# ---- Eq. 2 features --------------------------------
def test_phase_table_closed_forms():
    S, C = oracle.phase_table(48)
    assert abs(S[0]) < 1e-12 and abs(C[0] - 1) < 1e-12          # t=0  -> (0, 1)
    assert abs(S[12] - 1) < 1e-12 and abs(C[12]) < 1e-12        # t=12 -> (1, 0)
    assert abs(S[24]) < 1e-12 and abs(C[24] + 1) < 1e-12        # t=24 -> (0, -1)
    for T in (1, 4, 24, 48, 96, 288):
        S, C = oracle.phase_table(T)
        assert np.all(np.abs(S * S + C * C - 1.0) < 1e-9)
        # the table is the textbook function at the grid points
        ref = np.sin(2 * np.pi * np.arange(T) / T)
        assert np.max(np.abs(S - ref)) < 1e-15


# ---- exact rational pin (golden/fit_t4.json) --------------------
def test_fit_matches_exact_rational_least_squares():
    g = json.load(open(os.path.join(GOLDEN, "fit_t4.json")))
    hist = g["history"]
    m = oracle.fit(hist, T=g["T"], phi0=0)
    assert m.status == 0 and m.kind == 0 and m.n_cols == 3
    beta = [F(b) for b in g["beta_intercept_sin_cos_lag"]]
    # exact normal equations recomputed here, independent of the fixture
    sc = {0: (0, 1), 1: (1, 0), 2: (0, -1), 3: (-1, 0)}
    X = [[*sc[t % 4], hist[t - 1]] for t in range(1, len(hist))]
    assert exact.lstsq_intercept(X, hist[1:]) == beta
    got = [m.c0, m.ws, m.wc, m.wl]
    for a, b in zip(got, beta):
        assert abs(a - float(b)) <= 1e-9 * max(1.0, abs(float(b)))
    S, C = oracle.phase_table(4)
    chat = oracle.predict(m, S[6 % 4], C[6 % 4], 510.0)
    assert abs(chat - float(F(g["forecast_step6_lag510"]))) < 1e-9


@pytest.mark.parametrize("seed", range(12))
def test_fit_matches_numpy_lstsq(seed):
    """Random noisy diurnal histories: forecasts agree with SVD least squares."""
    rng = np.random.default_rng(seed)
    T = int(rng.choice([24, 48, 96]))
    L = int(rng.integers(6, 3 * T))
    phi0 = int(rng.integers(0, T))
    t = np.arange(L)
    hist = 500 + 150 * np.sin(2 * np.pi * (t + phi0 + rng.integers(0, T)) / T) + rng.normal(0, 20, L)
    hist = np.round(np.maximum(hist, 0) * 64) / 64
    m = oracle.fit(hist, T=T, phi0=phi0)
    assert m.status == 0 and m.kind == 0
    S, C = oracle.phase_table(T)
    rows = np.arange(1, L)
    X = np.column_stack([np.ones(L - 1), S[(phi0 + rows) % T], C[(phi0 + rows) % T], hist[rows - 1]])
    beta, *_ = np.linalg.lstsq(X, hist[rows], rcond=None)
    for phi in range(T):
        lag = float(hist[-1]) * (0.5 + phi / T)
        ref = beta[0] + beta[1] * S[phi] + beta[2] * C[phi] + beta[3] * lag
        got = oracle.predict(m, S[phi], C[phi], lag)
        assert abs(got - max(ref, 0.0)) <= 1e-9 * max(1.0, abs(ref))


def test_pure_sinusoid_in_sample_within_1e6():
    """target exactly A sin + B cos + C -> predictions within 1e-6.
    The lag column is then collinear with (sin, cos, 1): the ridge fires."""
    T, L = 24, 24
    S, C = oracle.phase_table(T)
    y = np.array([300 + 120 * S[t % T] - 45 * C[t % T] for t in range(L + 1)])
    m = oracle.fit(y[:L], T=T)
    assert m.status == 0 and m.ridge == 1
    for t in range(1, L + 1):
        got = oracle.predict(m, S[t % T], C[t % T], y[t - 1])
        assert abs(got - y[t]) <= 1e-6 * abs(y[t])


def test_constant_target_and_bias_only():
    """S:138 constant target 500 -> 500 everywhere; S:155 bias-only model."""
    m = oracle.fit([500.0] * 24, T=24)
    assert m.kind == 1 and m.status == 0
    S, C = oracle.phase_table(24)
    for phi in range(24):
        assert oracle.predict(m, S[phi], C[phi], 123.0 * phi) == 500.0
    # constant target with a varying first (lag-only) point is still constant
    m = oracle.fit([10.0] + [500.0] * 23, T=24)
    assert m.kind == 1 and oracle.predict(m, 0.3, 0.1, 99.0) == 500.0


def test_negative_prediction_clamps_to_zero():
    """S:157 / S:199: negative raw prediction -> 0."""
    m = oracle.Model()
    m.c0, m.ws, m.wc, m.wl = -50.0, 0.0, 0.0, 0.1
    assert oracle.predict(m, 0.0, 1.0, 100.0) == 0.0
    assert oracle.predict(m, 0.0, 1.0, 1000.0) == 50.0


def test_zero_variance_column_dropped():
    """S:114 / DESIGN Q7: with T=1 both phase features are constant; the fit is
    then a plain regression on the lag (exact rational pin)."""
    hist = [400.0, 500.0, 450.0, 350.0, 420.0, 510.0, 480.0]
    m = oracle.fit(hist, T=1)
    assert m.status == 0 and m.n_cols == 1 and m.ws == 0.0 and m.wc == 0.0
    b = exact.lstsq_intercept([[h] for h in hist[:-1]], hist[1:])
    assert abs(m.wl - float(b[1])) < 1e-12 and abs(m.c0 - float(b[0])) < 1e-9


def test_mape_linear_beats_persistence_on_synthetic_diurnal():
    """S:520 forecasting sanity (Table 1 not reproducible, P:156 trace not
    shipped): seeded diurnal trace, mean 550, amp 150, period 48, sigma 10,
    552 points, 24 h fit, walk-forward with the TRUE lag."""
    rng = np.random.default_rng(0)
    T, N, L = 48, 552, 48
    t = np.arange(N)
    c = 550 + 150 * np.sin(2 * np.pi * t / T) + rng.normal(0, 10, N)
    m = oracle.fit(c[:L], T=T)
    S, C = oracle.phase_table(T)
    pred = np.array([oracle.predict(m, S[w % T], C[w % T], c[w - 1]) for w in range(L, N)])
    act = c[L:]
    mape_lin = 100 * np.mean(np.abs(act - pred) / act)
    mape_per = 100 * np.mean(np.abs(act - c[L - 1:N - 1]) / act)
    assert mape_lin <= mape_per
    # noiseless sinusoid: linear MAPE < 0.1 %
    c0 = 550 + 150 * np.sin(2 * np.pi * t / T)
    m0 = oracle.fit(c0[:L], T=T)
    pred0 = np.array([oracle.predict(m0, S[w % T], C[w % T], c0[w - 1]) for w in range(L, N)])
    assert 100 * np.mean(np.abs(c0[L:] - pred0) / c0[L:]) < 0.1


def test_rolling_refit_uses_the_L_points_before_each_origin():
    """Rolling mode (Q1): window w with stride R refits on c[r-L, r)."""
    rng = np.random.default_rng(3)
    T, L, N = 24, 24, 24 + 50
    c = np.round((500 + 100 * np.sin(2 * np.pi * np.arange(N) / T) + rng.normal(0, 15, N)) * 64) / 64
    fc, ch, tot, st = oracle.plan_trace(c, L=L, T=T, refit_stride=7, avg_power=[100, 200], thr=[400, 700],
                                        etas=[0.5], pmax=300.0)
    assert st == 0
    S, C = oracle.phase_table(T)
    for w in (L, L + 6, L + 7, L + 20, N - 1):
        r = L + 7 * ((w - L) // 7)
        m = oracle.fit(c[r - L:r], T=T, phi0=(r - L) % T)
        assert fc[w - L] == oracle.predict(m, S[w % T], C[w % T], c[w - 1])


def test_rolling_refit_every_window_matches_numpy_lstsq():
    """R = 1 (a new model each window): every forecast equals
    SVD least squares (numpy, a different algorithm) on the L points before
    that window, clamped at 0."""
    rng = np.random.default_rng(12)
    T, L, N = 24, 24, 24 + 120
    t = np.arange(N)
    c = np.round((480 + 140 * np.sin(2 * np.pi * (t + 5) / T) + rng.normal(0, 18, N)) * 64) / 64
    fc, ch, tot, st = oracle.plan_trace(c, L=L, T=T, refit_stride=1, avg_power=[100, 200], thr=[400, 700],
                                        etas=[0.5], pmax=300.0)
    assert st == 0
    S, C = oracle.phase_table(T)
    for w in range(L, N):
        rows = np.arange(w - L + 1, w)
        X = np.column_stack([np.ones(L - 1), S[rows % T], C[rows % T], c[rows - 1]])
        beta, *_ = np.linalg.lstsq(X, c[rows], rcond=None)
        ref = beta[0] + beta[1] * S[w % T] + beta[2] * C[w % T] + beta[3] * c[w - 1]
        assert abs(fc[w - L] - max(ref, 0.0)) <= 1e-9 * max(1.0, abs(ref))
