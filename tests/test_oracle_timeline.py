"""Pins for timeline / audit emission (SPEC emit_timeline
S:413-421, SimReport invariants S:374-378 and S:424-426; Figure 1/2 rows,
PAPER.md:187-195): per-period rows of a planned fixed-work replay.
"""
import json
import os
from fractions import Fraction as F

import numpy as np
import pytest

import oracle
from oracle import exact
from conftest import GOLDEN


def test_golden_two_period_rows():
    """S:421 DERIVED: the corrected golden scenario gives 2 rows whose fields
    follow from hand integration (exact rationals), summing to the frozen totals."""
    g = json.load(open(os.path.join(GOLDEN, "golden_2period.json")))
    prof = g["profile"]
    c = [float(v) for v in g["trace"]]
    rows = oracle.timeline(np.array(c), L=0, choice=g["choices"], forecast=c, limit_w=prof["limit_w"],
                           avg_power=prof["avg_power_w"], thr=prof["throughput_sps"],
                           delta=float(g["interval_s"]), J=float(g["job_samples"]))
    assert rows.shape == (2, 8)
    d, J = F(g["interval_s"]), F(g["job_samples"])
    s1 = F(700) * d                                  # period 1: a full window at 200 W
    f2 = (J - s1) / (F(850) * d)                     # period 2: the completion fraction at 300 W
    want = [
        [0, 600, 600, 200, 190, s1, F(190) * d, F(190) * d * 600 / 3600000],
        [1, 50, 50, 300, 295, J - s1, f2 * 295 * d, f2 * 295 * d * 50 / 3600000],
    ]
    for r, wr in zip(rows, want):
        assert list(r[:5]) == [float(v) for v in wr[:5]]
        for a, b in zip(r[5:], wr[5:]):
            assert a == float(b)
    tot = [F(g["aware"]["energy_j"]), F(g["aware"]["carbon_g"])]
    assert rows[:, 6].sum() == float(tot[0]) and abs(rows[:, 7].sum() - float(tot[1])) < 1e-12
    assert rows[:, 5].sum() == float(J)              # work conservation


@pytest.mark.parametrize("seed,period", [(0, 1), (1, 7), (2, 24), (3, 5000)])
def test_rows_conserve_the_replay_totals(seed, period):
    """totals equal the sums of the period fields; samples sum to J;
    carbon per row is the stepwise integral (checked against exact rationals)."""
    rng = np.random.default_rng(seed)
    T, L, N = 24, 24, 24 + 400
    c = np.round((480 + 130 * np.sin(2 * np.pi * np.arange(N) / T) + rng.normal(0, 30, N)) * 64) / 64
    lim, P, Th = [150, 200, 250, 300], [140.0, 190.0, 238.0, 281.0], [400.0, 560.0, 680.0, 760.0]
    J = 3600 * 400 * 420.0
    fc, ch, tot, st = oracle.plan_trace(c, L=L, T=T, period=period, avg_power=P, thr=Th, etas=[0.6], pmax=300.0, J=J)
    assert st == 0
    rows = oracle.timeline(c, L=L, period=period, choice=ch[0], forecast=fc, limit_w=lim, avg_power=P, thr=Th, J=J)
    W = N - L
    assert len(rows) == -(-W // period)
    assert rows[:, 5].sum() == J
    assert abs(rows[:, 6].sum() - tot["energy_j"][0]) <= 1e-12 * tot["energy_j"][0]
    assert abs(rows[:, 7].sum() - tot["carbon_g"][0]) <= 1e-12 * tot["carbon_g"][0]
    ex = exact.replay(list(c), L, list(ch[0]), P, Th, 3600, J)
    assert abs(rows[:, 7].sum() - float(ex[2])) <= 1e-12 * float(ex[2])
    for j, r in enumerate(rows):                     # the period's own fields
        b = j * period
        seg = c[L + b:L + b + min(period, W - b)]
        assert r[0] == L + b and r[1] == fc[b] and abs(r[2] - seg.mean()) <= 1e-12 * seg.mean()
        assert r[3] == lim[ch[0][b]] and r[4] == P[ch[0][b]]


def test_baseline_rows_are_flat_at_the_max_limit():
    """the baseline report has a constant chosen_limit column (Figure 1's flat 300 W line)."""
    rng = np.random.default_rng(4)
    c = 400 + rng.random(24 + 50) * 100
    rows = oracle.timeline(c, L=24, period=1, choice=None, limit_w=[150, 300], avg_power=[140.0, 290.0],
                           thr=[400.0, 800.0], J=3600 * 30 * 800.0)
    assert np.all(rows[:, 3] == 300) and np.all(np.isnan(rows[:, 1]))
    assert rows[:30, 5].sum() == 3600 * 30 * 800.0 and np.all(rows[30:, 5:] == 0.0)
    one = oracle.timeline(c[:25], L=24, period=1, choice=None, limit_w=[150, 300], avg_power=[140.0, 290.0],
                          thr=[400.0, 800.0])
    assert one.shape == (1, 8)                       # S:419 one-period report -> one row


def test_eq3_summary_covariance_identity():
    """Eq. 3 vs the stepwise integration: over n full windows
    stepwise - Eq.3 = n * Cov(P, c) * Delta / 3.6e6 exactly (Cov the population
    covariance of the chosen power and the intensity); constant intensity makes
    them equal; aligned / anti-aligned power and intensity give the sign."""
    c = [500.0, 600.0, 200.0, 700.0, 100.0]            # L = 1: windows 600, 200, 700, 100
    lines = dict(avg_power=[100.0, 300.0], thr=[400.0, 800.0])
    for choice, sign in (([1, 0, 1, 0], 1), ([0, 1, 0, 1], -1)):
        out = oracle.job_summary(np.array(c), L=1, choice=choice, **lines)
        P = [lines["avg_power"][k] for k in choice]
        cw = c[1:]
        n = F(len(cw))
        cov = sum(F(p) * F(x) for p, x in zip(P, cw)) / n - (sum(map(F, P)) / n) * (sum(map(F, cw)) / n)
        assert out[0] - out[1] == float(n * cov * 3600 / 3600000)
        assert (out[0] - out[1]) * sign > 0
        assert out[2] == float(sum(map(F, P)) / n) and out[3] == float(sum(map(F, cw)) / n)
    flat = oracle.job_summary(np.full(9, 432.0), L=1, choice=[1, 0, 0, 1, 0, 1, 1, 0], **lines)
    assert flat[0] == flat[1] and flat[3] == 432.0


def test_eq3_summary_matches_the_replay_and_timeline():
    """The stepwise carbon is the replay's (and the timeline rows' sum); the
    energy behind Eq. 3 is the replay's energy; a completing job counts its
    last window pro rata (golden two-period scenario, exact rationals)."""
    g = json.load(open(os.path.join(GOLDEN, "golden_2period.json")))
    prof = g["profile"]
    c = np.array([float(v) for v in g["trace"]])
    out = oracle.job_summary(c, L=0, choice=g["choices"], avg_power=prof["avg_power_w"],
                             thr=prof["throughput_sps"], delta=float(g["interval_s"]), J=float(g["job_samples"]))
    d, J = F(g["interval_s"]), F(g["job_samples"])
    f2 = (J - F(700) * d) / (F(850) * d)               # completion fraction of window 2 at 300 W
    E = (F(190) + f2 * 295) * d                         # energy, J
    tw = 1 + f2
    avg_ci = (F(600) + f2 * 50) / tw
    assert abs(out[0] - float(F(g["aware"]["carbon_g"]))) <= 1e-12 * out[0]
    assert out[1] == float(E * avg_ci / 3600000) and out[3] == float(avg_ci)
    assert out[2] == float((F(190) + f2 * 295) / tw)
    rng = np.random.default_rng(7)
    T, L, N = 24, 24, 24 + 300
    tr = np.round((480 + 130 * np.sin(2 * np.pi * np.arange(N) / T) + rng.normal(0, 30, N)) * 64) / 64
    P, Th = [140.0, 190.0, 238.0, 281.0], [400.0, 560.0, 680.0, 760.0]
    J2 = 3600 * 250 * 420.0
    fc, ch, tot, st = oracle.plan_trace(tr, L=L, T=T, avg_power=P, thr=Th, etas=[0.6], pmax=300.0, J=J2)
    s = oracle.job_summary(tr, L=L, choice=ch[0], avg_power=P, thr=Th, J=J2)
    assert abs(s[0] - tot["carbon_g"][0]) <= 1e-12 * s[0]
    rows = oracle.timeline(tr, L=L, choice=ch[0], limit_w=[150, 200, 250, 300], avg_power=P, thr=Th, J=J2)
    assert abs(rows[:, 7].sum() - s[0]) <= 1e-12 * s[0]
    assert abs(s[2] * (tot["time_s"][0] / 3600) * 3600 - tot["energy_j"][0]) <= 1e-9 * tot["energy_j"][0]


def test_profiling_overhead_by_hand():
    """DESIGN Q33 (SPEC --count-profiling): K steps before the job, one
    per limit in increasing order, at each limit's average power."""
    c = np.array([100.0, 200.0, 300.0, 400.0, 500.0, 600.0])
    st, out = oracle.profiling_overhead(c, L=5, avg_power=[150.0, 250.0, 275.0], delta=1800.0)
    assert st == 0
    assert out[0] == 3 * 1800.0 and out[1] == (150 + 250 + 275) * 1800.0
    assert out[2] == float(F(150 * 300 + 250 * 400 + 275 * 500) * 1800 / 3600000)
    assert oracle.profiling_overhead(c, L=2, avg_power=[1.0, 2.0, 3.0])[0] == 2
