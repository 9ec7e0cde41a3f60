"""Pins for the forecast-evaluation sweep: SPEC mape
 and evaluate_models, the walk-forward Table 1
experiment of PAPER.md:159-161 on synthetic traces.
"""
import numpy as np
import pytest

import oracle


def test_mape_spec_examples():
    assert oracle.mape([100, 200], [110, 180]) == 10.0          # S:172, direct arithmetic
    a = np.array([120.0, 340.5, 77.25])
    assert oracle.mape(a, a) == 0.0                               # S:171 identity
    p = np.array([100.0, 300.0, 80.0])
    assert abs(oracle.mape(a * 8.0, p * 8.0) - oracle.mape(a, p)) <= 1e-12 * oracle.mape(a, p)  # scaling
    assert np.isnan(oracle.mape([100.0, 0.0], [90.0, 1.0]))        # S:171 zero actual
    # hand value: |100-90|/100 = 0.1, |50-60|/50 = 0.2 -> 15 %
    assert abs(oracle.mape([100.0, 50.0], [90.0, 60.0]) - 15.0) < 1e-12


def test_persistence_on_constant_trace_and_noiseless_sinusoid():
    st, lin, per = oracle.evaluate(np.full(100, 432.0), L=24, T=24)
    assert st == 0 and per == 0.0 and lin == 0.0
    t = np.arange(552)
    c = 550 + 150 * np.sin(2 * np.pi * t / 48)
    st, lin, per = oracle.evaluate(c, L=48, T=48)
    assert st == 0 and lin < 0.1 and per > 1.0                    # S:192 noiseless sinusoid


@pytest.mark.parametrize("seed", range(6))
def test_walk_forward_matches_numpy_least_squares(seed):
    """Linear MAPE equals an independent recomputation: numpy SVD least
    squares on the first L points, N-L one-step predictions with the true lag
    (the first seeded by the last fit point), numpy's MAPE."""
    rng = np.random.default_rng(seed)
    T = int(rng.choice([24, 48]))
    L = T * int(rng.integers(1, 3))
    N = L + int(rng.integers(50, 600))
    ph = int(rng.integers(0, T))
    t = np.arange(N)
    c = np.round((500 + 140 * np.sin(2 * np.pi * (t + ph) / T) + rng.normal(0, 25, N)) * 64) / 64
    st, lin, per = oracle.evaluate(c, L=L, T=T)
    assert st == 0
    S, C = oracle.phase_table(T)
    rows = np.arange(1, L)
    X = np.column_stack([np.ones(L - 1), S[rows % T], C[rows % T], c[rows - 1]])
    beta, *_ = np.linalg.lstsq(X, c[rows], rcond=None)
    w = np.arange(L, N)
    pred = np.maximum(beta[0] + beta[1] * S[w % T] + beta[2] * C[w % T] + beta[3] * c[w - 1], 0.0)
    ref = 100.0 * np.mean(np.abs(c[w] - pred) / c[w])
    assert abs(lin - ref) <= 1e-9 * ref
    ref_p = 100.0 * np.mean(np.abs(c[w] - c[w - 1]) / c[w])
    assert abs(per - ref_p) <= 1e-12 * ref_p
    assert lin <= per                                             # S:184 DERIVED direction


def test_paper_split_counts_and_statuses():
    """a 552-point trace fitted on 48 points gives 504 predictions."""
    rng = np.random.default_rng(0)
    c = 550 + 150 * np.sin(2 * np.pi * np.arange(552) / 48) + rng.normal(0, 10, 552)
    st, lin, per = oracle.evaluate(c, L=48, T=48)
    assert st == 0
    ref_p = 100.0 * np.mean(np.abs(c[48:] - c[47:-1]) / c[48:])   # 504 terms
    assert len(c[48:]) == 504 and abs(per - ref_p) <= 1e-12 * ref_p
    bad = c.copy()
    bad[100] = -1.0
    assert oracle.evaluate(bad, L=48, T=48)[0] == 4
    zero = c.copy()
    zero[300] = 0.0
    st, lin, per = oracle.evaluate(zero, L=48, T=48)
    assert st == 8 and np.isnan(lin)
    out, sts, _ = oracle.evaluate_batch(np.stack([c, bad, zero]).astype(np.float32), N=552, L=48, T=48)
    assert list(sts) == [0, 4, 8]
