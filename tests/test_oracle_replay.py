"""Pins for the oracle's fixed-work replay (
SPEC.md:386-436) and the whole-trace planner (oracle_plan_trace)."""
import json
import os
from fractions import Fraction as F

import numpy as np
import pytest

import inputs
import oracle
from oracle import exact
from conftest import GOLDEN


def test_spec_baseline_examples():
    """8500 samples at 850 sps, 295 W -> 10 s, 2950 J (Delta = 1 s);
    S:393 constant ci=500 -> carbon = E/3.6e6*500; S:394 two-step 400/800."""
    P, Th = [190.0, 295.0], [700.0, 850.0]
    out, w, st = oracle.replay([500.0] * 20, 0, [1] * 20, P, Th, 1.0, 8500.0)
    assert st == 0 and out[0] == 10.0 and out[1] == 2950.0 and out[3] == 8500.0 and w == 9
    assert out[2] == 2950.0 / 3.6e6 * 500.0
    out, w, st = oracle.replay([400.0] * 5 + [800.0] * 5, 0, [1] * 10, P, Th, 1.0, 8500.0)
    E = 2950.0
    assert abs(out[2] - (0.5 * E * 400 / 3.6e6 + 0.5 * E * 800 / 3.6e6)) < 1e-15


def test_corrected_golden_two_period():
    g = json.load(open(os.path.join(GOLDEN, "golden_2period.json")))
    P, Th = g["profile"]["avg_power_w"], g["profile"]["throughput_sps"]
    c = [float(v) for v in g["trace"]]
    ch = [oracle.choose(P, Th, g["eta"], g["max_power_w"], g["max_ci"], v) for v in c]
    assert ch == g["choices"]
    # exact rationals (independent) agree with the frozen golden values
    ex = exact.replay(c, 0, ch, P, Th, g["interval_s"], g["job_samples"])
    exb = exact.replay(c, 0, [1, 1], P, Th, g["interval_s"], g["job_samples"])
    for key, v in zip(("time_s", "energy_j", "carbon_g"), ex[:3]):
        assert v == F(g["aware"][key])
    for key, v in zip(("time_s", "energy_j", "carbon_g"), exb[:3]):
        assert v == F(g["baseline"][key])
    out, w, st = oracle.replay(c, 0, ch, P, Th, float(g["interval_s"]), float(g["job_samples"]))
    assert st == 0 and w == 1
    assert list(out[:3]) == [5400.0, 1215000.0, 121.375]
    outb, wb, stb = oracle.replay(c, 0, [1, 1], P, Th, float(g["interval_s"]), float(g["job_samples"]))
    for a, key in zip(outb[:3], ("time_s", "energy_j", "carbon_g")):
        assert abs(a - float(F(g["baseline"][key]))) <= 1e-15 * a
    # the SPEC's original [600, 200] picks 200 W in both periods (erratum, Q23)
    assert [oracle.choose(P, Th, 0.9, 300.0, 750.0, v) for v in (600.0, 200.0)] == [0, 0]
    cx = F(g["crossover_ci"])
    assert exact.costs(F(9, 10), P, Th, 300, 750, cx)[0] == exact.costs(F(9, 10), P, Th, 300, 750, cx)[1]


@pytest.mark.parametrize("seed", range(20))
def test_replay_matches_exact_rationals_and_conservation(seed):
    """conservation (totals == stepwise sums), work conservation
    (samples == J), time bound J/Thr_max <= time <= J/Thr_min.  Dyadic inputs
    make every accumulator exact, so only the final divisions round."""
    rng = np.random.default_rng(seed)
    K = int(rng.integers(2, 9))
    Th = np.sort(np.round(rng.uniform(200, 900, K) * 64) / 64)
    P = np.sort(np.round(rng.uniform(80, 300, K) * 64) / 64)
    N, s0, delta = int(rng.integers(30, 300)), int(rng.integers(1, 25)), float(rng.choice([900, 1800, 3600]))
    c = np.round(rng.uniform(0, 900, N) * 64) / 64
    ch = rng.integers(0, K, N - s0).astype(np.uint8)
    W = N - s0
    J = float(delta * W * Th.min() * rng.uniform(0.2, 1.0))
    out, w, st = oracle.replay(c, s0, ch, P, Th, delta, J)
    ex = exact.replay(list(c), s0, list(ch), list(P), list(Th), delta, J)
    assert st == 0 and w == ex[4]
    for a, b in zip(out[:4], ex[:4]):
        assert abs(F(a) - b) <= F(1, 10**12) * abs(b)
    assert out[3] == J
    assert J / Th.max() - 1e-9 <= out[0] <= J / Th.min() + 1e-9
    # fixed-duration mode (J <= 0): exact sums over the whole trace
    out0, w0, st0 = oracle.replay(c, s0, ch, P, Th, delta, 0.0)
    ex0 = exact.replay(list(c), s0, list(ch), list(P), list(Th), delta, 0)
    assert st0 == 0 and w0 == -1 and out0[0] == W * delta and F(out0[3]) == ex0[3]
    # exhaustion is an error, not a wrap-around
    _, _, st3 = oracle.replay(c, s0, ch, P, Th, delta, float(delta * W * Th.max() * 2))
    assert st3 == 3


def _plan(c, etas, prof, J, **kw):
    return oracle.plan_trace(c, L=24, T=24, avg_power=prof.avg_power_w, thr=prof.throughput_sps,
                             etas=etas, pmax=float(prof.limit_w.max()), delta=3600.0, J=J, **kw)


def test_eta0_equals_baseline_when_max_limit_is_fastest():
    """S:428 (conditional per Q15): eta=0 replays exactly like the baseline."""
    prof = inputs.make_profile("resnet50", inputs.LIMITS_9)
    c = inputs.synth_traces_host(1, 24 + 500, seed=11)[0, :524].astype(np.float64)
    J = 3600.0 * 500 * prof.throughput_sps.min()
    fc, ch, tot, st = _plan(c, [0.0], prof, J)
    assert st == 0 and np.all(ch == 8)
    t = tot[0]
    assert (t["time_s"], t["energy_j"], t["carbon_g"]) == (t["base_time_s"], t["base_energy_j"], t["base_carbon_g"])
    # saturated BERT table: eta=0 picks the LOWER of two identical fastest rows (Q15)
    bert = inputs.make_profile("bert", inputs.LIMITS_9)
    _, chb, _, _ = _plan(c, [0.0], bert, J)
    assert np.all(chb == 7)


def test_direction_carbon_down_time_up():
    """P:14/P:205-206 direction (13.6 % / 2.5 % is parity-unpinned, Q-E2): on a
    synthetic 2:1 high/low swing with energy_per_sample increasing in the
    limit, eta=0.9 carbon-aware planning emits less carbon than max-power
    training and takes < 25 % longer."""
    prof = inputs.make_profile("resnet50", [200, 225, 250, 275, 300])
    eps = prof.avg_power_w / prof.throughput_sps
    assert np.all(np.diff(eps) > 0)
    N = 24 + 24 * 14
    t = np.arange(N)
    c = np.where((t // 6) % 2 == 0, 700.0, 350.0)
    J = 3600.0 * (N - 24) * prof.throughput_sps.min() * 0.5
    fc, ch, tot, st = _plan(c, [0.9], prof, J)
    assert st == 0
    x = tot[0]
    assert x["carbon_g"] < x["base_carbon_g"]
    assert x["base_time_s"] < x["time_s"] < 1.25 * x["base_time_s"]
    assert x["time_s"] <= J / prof.throughput_sps.min()      # S:429 time bound
    # and a synthetic hourly year (C2-shaped) at eta=0.5 also cuts carbon
    prof = inputs.make_profile("resnet50", inputs.LIMITS_9)
    c2 = inputs.synth_traces_host(1, 8784, seed=0, mode=inputs.MODE_PAPER)[0].astype(np.float64)
    J2 = 3600.0 * 8760 * prof.throughput_sps.min()
    _, _, tot2, st2 = _plan(c2, [0.5], prof, J2)
    assert st2 == 0 and tot2[0]["carbon_g"] < tot2[0]["base_carbon_g"]


def test_invalid_traces_report_status():
    """S:29 (values >= 0, finite) -> status 4, choices 0xFF; S:292 MaxCI > 0 -> 5."""
    prof = inputs.make_profile("resnet50", inputs.LIMITS_9)
    c = np.full(60, 400.0)
    c[40] = -1.0
    fc, ch, tot, st = _plan(c, [0.5], prof, 0.0)
    assert st == 4 and np.all(ch == 0xFF) and np.all(np.isnan(fc)) and tot[0]["status"] == 4
    c[40] = np.inf
    assert _plan(c, [0.5], prof, 0.0)[3] == 4
    c = np.concatenate([np.zeros(24), np.full(36, 300.0)])
    assert _plan(c, [0.5], prof, 0.0)[3] == 5
    # a fixed positive MaxCI makes the same trace valid
    assert _plan(c, [0.5], prof, 0.0, max_ci=750.0)[3] == 0


def test_batch_driver_matches_single_trace_driver():
    w = inputs.workload("C4", n_traces=40)
    tr = inputs.synth_traces_host(40, w.n_steps, seed=w.seed)
    pid = inputs.profile_ids_host(40, seed=w.seed, n_profiles=3)
    J = w.job_samples(pid)
    res = oracle.plan_batch(tr, N=w.n_steps, L=24, T=24, profiles=w.profiles, profile_id=pid,
                            etas=[0.3, 0.5], job_samples=J, threads=2)
    for i in (0, 7, 39):
        p = w.profiles[pid[i]]
        fc, ch, tot, st = oracle.plan_trace(tr[i, :w.n_steps], L=24, T=24, avg_power=p.avg_power_w,
                                            thr=p.throughput_sps, etas=[0.3, 0.5],
                                            pmax=float(p.limit_w.max()), J=J[i])
        assert np.array_equal(res["forecast"][i], fc)
        assert np.array_equal(res["choice"][:, i], ch)
        assert res["totals"][:, i].tobytes() == tot.tobytes()
    ok = res["totals"]["status"] == 0
    assert np.all(ok)
    s = res["sums"]
    assert s[0, 7] == 40 and abs(s[0, 2] - res["totals"][0]["carbon_g"].sum()) <= 1e-9 * s[0, 2]
