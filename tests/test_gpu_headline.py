"""GPU parity of the kernel bench.py times: sweep_fast_kernel<0> (fp32 traces,
16-byte aligned job start, one eta, no forecast output), against the oracle,
on the method's edge cases (VERDICT r1 "What's missing" 5, "What's weak" 2-3).

Every test asserts through chase_diag_t.kernel_path that the headline kernel
is the one that ran.  Bars (BASELINE.json north_star): choices bit-exact,
totals bit-identical for dyadic inputs and <= 1e-9 relative otherwise.

  - adversarial Eq. 6 bands: constant histories make the forecast exactly the
    constant (F2), so stepping MaxPower (per-trace MaxCI)
    or a fixed MaxCI by +-300 ulps walks every window's Eq. 6 key across each
    envelope breakpoint of the ResNet-shaped table;
  - eta = 0 and eta = 1 in a single-eta call;
  - fixed MaxCI / MaxPower;
  - raw forecasts below zero, clamped to 0 (Q8);
  - the SPEC 3-row exact tie at chat = 750;
  - non-dyadic traces and profiles, including a budget J that equals the
    oracle's running sum exactly (Q22).
"""
from fractions import Fraction as F

import numpy as np
import pytest

import inputs
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2303_02508_b200 as cb  # noqa: E402

DEV = torch.device("cuda:0")
RESNET = inputs.make_profile("resnet50", inputs.LIMITS_9)


def gpu_plan(tr, N, profiles, eta, *, pid=None, J=None, L=24, max_ci=0.0, max_power_w=0.0, dtype=torch.float32,
             expect=cb.PATH_HEADLINE, period=0):
    x = torch.from_numpy(np.ascontiguousarray(tr)).to(DEV, dtype)
    pl = cb.Planner(x, n_steps=N, profiles=profiles, etas=[eta], history_len=L,
                    profile_id=None if pid is None else torch.from_numpy(np.ascontiguousarray(pid, np.uint8)).to(DEV),
                    job_samples=None if J is None else torch.from_numpy(np.ascontiguousarray(J, np.float64)).to(DEV),
                    want_choice=True, want_forecast=False, want_per_trace=True, max_ci=max_ci,
                    max_power_w=max_power_w, period_steps=period)
    res = pl.run()
    torch.cuda.synchronize()
    d = pl.diag()
    assert d.kernel_path & expect, f"kernel_path={d.kernel_path:#x}: expected {expect:#x}"
    return dict(choice=res.choice.cpu().numpy()[0, :, :N - L], totals=res.per_trace_numpy()[0],
                sums=res.sums.cpu().numpy()[0], diag=d)


def oracle_plan(tr, N, profiles, eta, *, pid=None, J=None, L=24, max_ci=0.0, max_power_w=0.0, period=0):
    o = oracle.plan_batch(np.ascontiguousarray(tr, np.float32), N=N, L=L, T=24, profiles=profiles, profile_id=pid,
                          etas=[eta], pmax=max_power_w, max_ci=max_ci, job_samples=J, period=period)
    return dict(choice=o["choice"][0], totals=o["totals"][0], sums=o["sums"][0])


FIELDS = ("time_s", "energy_j", "carbon_g", "samples", "base_time_s", "base_energy_j", "base_carbon_g")


def assert_same(g, o, *, exact=True):
    bad = np.argwhere(g["choice"] != o["choice"])
    assert len(bad) == 0, f"{len(bad)} choice mismatches, first {tuple(bad[0])}: " \
                          f"gpu {g['choice'][tuple(bad[0])]} oracle {o['choice'][tuple(bad[0])]}"
    gt, ot = g["totals"], o["totals"]
    assert np.array_equal(gt["status"], ot["status"])
    assert np.array_equal(gt["completion_window"], ot["completion_window"])
    for f in FIELDS:
        if exact:
            assert np.array_equal(gt[f], ot[f]), f
        else:
            np.testing.assert_allclose(gt[f], ot[f], rtol=1e-9, atol=0, err_msg=f)
    np.testing.assert_allclose(g["sums"], o["sums"], rtol=1e-9, atol=1e-300)


def breakpoints(profile, eta):
    """Exact envelope breakpoints y* (in y = chat/Kc) of cost_k = (a_k y + 1)/Thr_k,
    a_k = eta P_k (Eq. 6 divided by Kc), with their line pair."""
    P = [F(float(v)) for v in profile.avg_power_w]
    Th = [F(float(v)) for v in profile.throughput_sps]
    e = F(eta)
    a = [e * v for v in P]
    K = len(P)
    out = []
    for j in range(K):
        for k in range(j + 1, K):
            den = a[k] * Th[j] - a[j] * Th[k]
            if den == 0:
                continue
            y = (Th[k] - Th[j]) / den
            if y <= 0:
                continue
            c = [(a[m] * y + 1) / Th[m] for m in range(K)]
            if c[j] == min(c) and c[k] == min(c):
                out.append((y, j, k))
    return sorted(out)


def constant_history_traces(values, N, L=24, seed=0):
    """fp32 traces whose L history points all equal v (the fit is the constant
    model, chat = v in every window, F2) and whose windows vary (the replay)."""
    rng = np.random.default_rng(seed)
    ld = inputs.round_up(N, 4)
    tr = np.zeros((len(values), ld), np.float32)
    for i, v in enumerate(values):
        tr[i, :L] = np.float32(v)
        tr[i, L:N] = rng.uniform(50.0, 900.0, N - L).astype(np.float32)
    return tr


def ulp_steps(x0, n):
    xs, x = [], float(x0)
    for _ in range(n):
        x = float(np.nextafter(x, -np.inf))
    for _ in range(2 * n + 1):
        xs.append(x)
        x = float(np.nextafter(x, np.inf))
    return xs


# ------------------------------------------------------------------ adversarial Eq. 6 bands
@pytest.mark.parametrize("eta", [0.9, 0.7])
def test_headline_band_sweep_max_power(eta):
    """Per-trace MaxCI = v (the constant history), so y = v/((1-eta) Pmax v)
    ~ 1/((1-eta) Pmax) for every trace and window: Pmax* = 1/((1-eta) y*) puts
    each reachable breakpoint y* (Pmax* >= 300 W, the largest limit) under
    every window; +-300 ulps of Pmax walk the key across its rounding band.
    The 24 constants give different roundings of y at each step."""
    N = 24 + 1940       # one full warp chunk (1920 windows) and a ragged last chunk
    vals = [np.float32(97.0 + 31.713 * i) for i in range(24)]
    tr = constant_history_traces(vals, N)
    slow = 0
    bps = [(y, j, k) for (y, j, k) in breakpoints(RESNET, eta) if 1 / ((1 - F(eta)) * y) >= 300]
    assert len(bps) >= 6
    for y, j, k in bps:
        pm0 = float(1 / ((1 - F(eta)) * y))
        for pm in ulp_steps(pm0, 300):
            g = gpu_plan(tr, N, [RESNET], eta, max_power_w=pm)
            o = oracle_plan(tr, N, [RESNET], eta, max_power_w=pm)
            assert_same(g, o, exact=False)
            slow += g["diag"].n_slow_windows
    assert slow > 0, "no window reached the canonical rule: the band was not hit"


@pytest.mark.parametrize("period", [3, 24, 168])
def test_periods_band_sweep_max_power(period):
    """The MaxPower band sweep with decision periods: constant
    histories give A = v, w_lag = 0, so each period's horizon mean is v and
    the closed-form mean fl(fl(P v) fl(1/P)) lands within an ulp
    of it.  Pmax walks +-300 ulps around every breakpoint (keys inside the
    band the hi32 bucket test leaves, 2^-20 relative: sequential horizon,
    canonical rule) and then +-3 * 2^-20 in steps of 2^-20/20 (keys crossing
    the band's edges, where the envelope's 2^-36 shrink decides which keys
    the closed form may take).  P = 3: lane-local periods (PM 5), 24: per-chunk
    chains (PM 1), 168: 32-period batches (PM 2)."""
    eta = 0.9
    N = 24 + 1940
    vals = [np.float32(97.0 + 31.713 * i) for i in range(24)]
    tr = constant_history_traces(vals, N)
    slow = seq = calls = 0
    bps = [(y, j, k) for (y, j, k) in breakpoints(RESNET, eta) if 1 / ((1 - F(eta)) * y) >= 300]
    for y, j, k in bps:
        pm0 = float(1 / ((1 - F(eta)) * y))
        pms = ulp_steps(pm0, 300)[::6] + [pm0 * (1 + d * 2.0 ** -20) for d in np.linspace(-3, 3, 121)]
        for pm in pms:
            g = gpu_plan(tr, N, [RESNET], eta, max_power_w=pm, period=period, expect=cb.PATH_H_PERIODS)
            o = oracle_plan(tr, N, [RESNET], eta, max_power_w=pm, period=period)
            assert_same(g, o, exact=False)
            slow += g["diag"].n_slow_windows
            seq += g["diag"].n_seq_periods
            calls += 1
    full = calls * len(vals) * ((N - 24) // period)
    assert slow > 0, "no period reached the canonical rule: the band was not hit"
    assert seq < 0.9 * full, f"the closed form decided almost nothing ({seq} of {full} periods sequential)"
    assert seq > 0


def test_headline_band_sweep_fixed_max_ci():
    """Fixed MaxCI: y = v/((1-eta) 300 MaxCI); MaxCI* puts breakpoint
    y* exactly at the constant v = 750; +-300 ulps of MaxCI per breakpoint of
    the eta = 0.5 envelope (all eight), the other 15 traces nearby in fp32."""
    eta, v0 = 0.5, np.float32(750.0)
    N = 24 + 64
    vals = [v0] + [np.float32(v0 * (1 + d * 2.0 ** -23)) for d in range(-7, 8) if d]
    tr = constant_history_traces(vals, N, seed=1)
    slow = 0
    for y, j, k in breakpoints(RESNET, eta):
        mc0 = float(F(float(v0)) / ((1 - F(eta)) * 300 * y))
        for mc in ulp_steps(mc0, 300):
            g = gpu_plan(tr, N, [RESNET], eta, max_ci=mc)
            o = oracle_plan(tr, N, [RESNET], eta, max_ci=mc)
            assert_same(g, o, exact=False)
            slow += g["diag"].n_slow_windows
    assert slow > 0


def test_headline_spec_exact_tie_at_750():
    """SPEC 3-row table, eta 0.5, Pmax 300, chat = MaxCI = 750 exactly: cost(200 W)
    = 525/2 = cost(300 W), exact in fp64 -> first minimum, 200 W (index 1)."""
    prof = inputs.Profile("spec3", np.array([100, 200, 300], np.int32), np.array([105.0, 190.0, 295.0]),
                          np.array([400.0, 700.0, 850.0]))
    N = 24 + 200
    tr = constant_history_traces([750.0] * 5, N, seed=2)
    g = gpu_plan(tr, N, [prof], 0.5)
    o = oracle_plan(tr, N, [prof], 0.5)
    assert np.all(o["choice"] == 1)
    assert_same(g, o, exact=False)
    assert g["diag"].n_slow_windows == 5 * 200   # every window sits on the tie: all canonical


# ------------------------------------------------------------------ eta, MaxCI, clamp
@pytest.mark.parametrize("eta", [0.0, 1.0])
def test_headline_eta_0_and_1(eta):
    """eta = 0 (throughput only) and eta = 1 (carbon only, Kc = 0: y = x) in a
    single-eta call, C4-shaped (three profile shapes, BERT's tied rows)."""
    w = inputs.workload("C4", n_traces=257)
    N = 24 + 3000
    tr = inputs.synth_traces_host(w.n_traces, N, seed=w.seed)
    pid = inputs.profile_ids_host(w.n_traces, seed=w.seed, n_profiles=3)
    J = np.array([3600.0 * (N - 24) * float(w.profiles[p].throughput_sps.min()) for p in pid])
    g = gpu_plan(tr, N, w.profiles, eta, pid=pid, J=J)
    o = oracle_plan(tr, N, w.profiles, eta, pid=pid, J=J)
    assert_same(g, o)
    if eta == 0.0:   # argmax Thr, lowest index on ties (BERT: 275 W == 300 W)
        for p in range(3):
            thr = w.profiles[p].throughput_sps
            assert np.all(g["choice"][pid == p] == int(np.argmax(thr)))


@pytest.mark.parametrize("max_ci,max_power_w", [(600.0, 0.0), (1e4, 0.0), (35.5, 0.0), (750.0, 410.0), (0.0, 355.0)])
def test_headline_fixed_max_ci_and_max_power(max_ci, max_power_w):
    w = inputs.workload("C5", n_traces=300)
    N = 24 + 2500
    tr = inputs.synth_traces_host(w.n_traces, N, seed=9)
    J = np.full(w.n_traces, 3600.0 * (N - 24) * float(RESNET.throughput_sps.min()))
    g = gpu_plan(tr, N, [RESNET], 0.5, J=J, max_ci=max_ci, max_power_w=max_power_w)
    o = oracle_plan(tr, N, [RESNET], 0.5, J=J, max_ci=max_ci, max_power_w=max_power_w)
    assert_same(g, o)


def test_headline_negative_raw_forecast_clamps_to_zero():
    """An alternating history fits w_lag ~ -1 with c0 ~ 2 mean, so a window after
    a large value forecasts below zero: chat = max(0, .) = 0 (Q8).  The
    kernel looks up the unclamped key (negative y, bucket 0); it must decide
    like chat = 0."""
    rng = np.random.default_rng(5)
    n, N = 40, 24 + 700
    tr = np.zeros((n, N), np.float32)
    for i in range(n):
        base = 200.0 + 10.0 * i
        hist = np.where(np.arange(24) % 2 == 0, base - 90.0, base + 90.0) + rng.uniform(-3, 3, 24)
        tr[i, :24] = np.round(hist * 64) / 64
        win = rng.uniform(50.0, 400.0, N - 24)
        win[rng.random(N - 24) < 0.2] = 3000.0 + 100.0 * rng.random()   # spikes -> negative raw forecasts
        tr[i, 24:] = np.round(win * 64) / 64
    # the oracle's raw forecasts do go negative here
    m = oracle.fit(tr[0, :24].astype(np.float64), T=24)
    assert m.wl < -0.5
    assert m.c0 + m.wl * 3000.0 < 0.0
    g = gpu_plan(tr, N, [RESNET], 0.5)
    o = oracle_plan(tr, N, [RESNET], 0.5)
    assert_same(g, o)
    fc, ch, _, _ = oracle.plan_trace(tr[0, :N].astype(np.float64), L=24, T=24, avg_power=RESNET.avg_power_w,
                                     thr=RESNET.throughput_sps, etas=[0.5], pmax=300.0)
    assert np.any(fc == 0.0)


# ------------------------------------------------------------------ non-dyadic inputs
def nondyadic_profile(seed=0):
    """The ResNet-shaped table with arbitrary decimals added (not multiples of
    1/64), so the argmin still sweeps the limits."""
    rng = np.random.default_rng(seed)
    thr = RESNET.throughput_sps * (1.0 + 1e-3 * rng.random(RESNET.K)) + 1e-6 * rng.random(RESNET.K)
    pw = RESNET.avg_power_w - 0.37 * rng.random(RESNET.K) - 1e-7 * rng.random(RESNET.K)
    return inputs.Profile("nondyadic", RESNET.limit_w.copy(), pw, np.sort(thr))


def nondyadic_traces(n, N, seed=0):
    rng = np.random.default_rng(seed)
    t = np.arange(N)
    mean = rng.uniform(150.0, 700.0, (n, 1))
    amp = rng.uniform(0.05, 0.3, (n, 1)) * mean
    v = mean + amp * np.sin(2 * np.pi * (t + rng.integers(0, 24, (n, 1))) / 24) + rng.normal(0, 0.03, (n, N)) * mean
    return np.maximum(v, 1.0) * (1.0 + 1e-7 * rng.random((n, N)))   # arbitrary decimals


def test_nondyadic_headline_fp32():
    """Non-dyadic fp32 traces and profile: the headline's reordered (pairwise)
    replay sums differ from the oracle's sequential ones by rounding, so totals
    agree to 1e-9 and choices stay bit-exact (identical forecasts)."""
    n, N = 300, 24 + 4000
    prof = nondyadic_profile(1)
    tr = nondyadic_traces(n, inputs.round_up(N, 4), seed=2).astype(np.float32)
    J = np.full(n, 3600.0 * (N - 24) * float(prof.throughput_sps.min()) * 0.97)
    g = gpu_plan(tr, N, [prof], 0.5, J=J)
    o = oracle_plan(tr, N, [prof], 0.5, J=J)
    assert_same(g, o, exact=False)
    assert np.all(o["totals"]["completion_window"] > 0)


def shaped_traces(n, N, seed=0):
    """Non-dyadic fp32 traces of varied shape for the closed-form period
    horizons: deep diurnal swings (some phases' A(phi) < 0),
    near-persistent random walks (w_lag near 1), anti-persistent noise
    (w_lag < 0), near-constant traces and intensities close to zero."""
    rng = np.random.default_rng(seed)
    t = np.arange(N)
    out = np.empty((n, N))
    for i in range(n):
        kind = i % 5
        mean = rng.uniform(50.0, 600.0)
        if kind == 0:     # persistent (AR(1)) with a deep diurnal forcing: A(phi) < 0 at some phases
            ph, phi = rng.integers(0, 24), rng.uniform(0.6, 0.9)
            force = mean * (1.0 + 0.9 * np.sin(2 * np.pi * (t + ph) / 24)) + rng.normal(0, 0.01 * mean, N)
            v = np.empty(N)
            v[0] = mean
            for k in range(1, N):
                v[k] = phi * v[k - 1] + (1.0 - phi) * force[k]
        elif kind == 1:   # random walk around the mean
            v = mean + np.cumsum(rng.normal(0, 0.02 * mean, N))
        elif kind == 2:   # alternating noise (negative lag coefficient)
            v = mean + 0.2 * mean * (-1.0) ** t * rng.uniform(0.5, 1.0, N)
        elif kind == 3:   # near-constant
            v = mean + rng.normal(0, 1e-3, N)
        else:             # small intensities
            v = rng.uniform(0.5, 3.0) * (1.0 + 0.5 * np.sin(2 * np.pi * t / 24)) + rng.normal(0, 0.05, N)
        out[i] = v
    return np.maximum(out, 0.01) * (1.0 + 1e-7 * rng.random((n, N)))


@pytest.mark.parametrize("P", [2, 3, 5, 12, 24, 48, 168, 720])
def test_periods_shaped_nondyadic_traces(P):
    """Decision periods on non-dyadic traces of every shape the closed-form
    horizon has to handle or decline (clamped horizons, |w_lag| near 1,
    w_lag < 0, tiny means): choices bit-exact, totals within 1e-9 of the
    oracle, through the headline kernel's period paths."""
    n, N = 200, 24 + 3000
    prof = nondyadic_profile(3)
    tr = shaped_traces(n, inputs.round_up(N, 4), seed=P).astype(np.float32)
    # (a budget off every whole number of min-throughput windows: near-constant traces pick
    # one limit throughout, and J = m s_k exactly would be the S == J tie of Q22)
    J = np.full(n, 3600.0 * (N - 24) * float(prof.throughput_sps.min()) * 0.9 * (1.0 + 3.1e-7))
    g = gpu_plan(tr, N, [prof], 0.5, J=J, period=P, expect=cb.PATH_H_PERIODS)
    o = oracle_plan(tr, N, [prof], 0.5, J=J, period=P)
    assert_same(g, o, exact=False)


def _oracle_running_samples(choice, thr, delta):
    """S after each window in the oracle's sequential order (R1: S += Thr_k*Delta)."""
    s, out = 0.0, []
    for k in choice:
        s = s + float(thr[k]) * delta
        out.append(s)
    return out


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_nondyadic_budget_equal_to_running_sum(dtype):
    """J equal to the oracle's running sum S at a window (S == J, Q22): the
    oracle completes there with f = 1; the GPU's differently ordered sum may
    land one rounding below J and complete at the next window with f ~ 0.
    Both give the same totals (to 1e-9): accept either completion window."""
    n, N = 64, 24 + 2100
    prof = nondyadic_profile(3)
    tr64 = nondyadic_traces(n, inputs.round_up(N, 4), seed=4)
    tr = tr64.astype(np.float32) if dtype == torch.float32 else tr64
    o0 = None
    J = np.zeros(n)
    for i in range(n):
        c = tr[i, :N].astype(np.float64)
        fc, ch, tot, st = oracle.plan_trace(c, L=24, T=24, avg_power=prof.avg_power_w, thr=prof.throughput_sps,
                                           etas=[0.5], pmax=300.0)
        S = _oracle_running_samples(ch[0], prof.throughput_sps, 3600.0)
        J[i] = S[700 + 17 * i]
    exp_path = cb.PATH_HEADLINE if dtype == torch.float32 else cb.PATH_GENERAL
    g = gpu_plan(tr, N, [prof], 0.5, J=J, dtype=dtype, expect=exp_path)
    for i in range(n):
        c = tr[i, :N].astype(np.float64)
        fc, ch, tot, st = oracle.plan_trace(c, L=24, T=24, avg_power=prof.avg_power_w, thr=prof.throughput_sps,
                                           etas=[0.5], pmax=300.0, J=float(J[i]))
        assert tot[0]["completion_window"] == 24 + 700 + 17 * i
        assert np.array_equal(g["choice"][i], ch[0])
        gw = int(g["totals"]["completion_window"][i])
        assert gw in (tot[0]["completion_window"], tot[0]["completion_window"] + 1), (i, gw)
        for f in FIELDS:
            np.testing.assert_allclose(g["totals"][f][i], tot[0][f], rtol=1e-9, atol=1e-9, err_msg=f)


def test_headline_smem_limit_falls_back_to_general_kernel():
    """5-minute data (T = 288) and 8 profiles at T = 24 exceed one CTA's shared
    memory in the headline layout: the general kernel takes them."""
    rng = np.random.default_rng(7)
    # T = 288, L = 288: one trace of 3 days
    N = 288 + 600
    tr = inputs.synth_traces_host(3, N, seed=11, T=288)
    J = np.full(3, 300.0 * 600 * float(RESNET.throughput_sps.min()))
    x = torch.from_numpy(tr).to(DEV)
    pl = cb.Planner(x, n_steps=N, profiles=[RESNET], etas=[0.5], interval_s=300, history_len=288,
                    job_samples=torch.from_numpy(J).to(DEV), want_choice=True, want_per_trace=True)
    res = pl.run()
    torch.cuda.synchronize()
    assert pl.diag().kernel_path & cb.PATH_GENERAL
    o = oracle.plan_batch(tr, N=N, L=288, T=288, profiles=[RESNET], etas=[0.5], delta=300.0, job_samples=J)
    assert np.array_equal(res.choice.cpu().numpy()[0, :, :N - 288], o["choice"][0])
    # 8 profiles at T = 24
    profs = [inputs.make_profile(s, inputs.LIMITS_9) for s in ("resnet50", "bert", "vit")] * 3
    profs = profs[:8]
    n, N = 200, 24 + 500
    tr = inputs.synth_traces_host(n, N, seed=12)
    pid = rng.integers(0, 8, n).astype(np.uint8)
    g = gpu_plan(tr, N, profs, 0.5, pid=pid, expect=cb.PATH_GENERAL)
    o = oracle_plan(tr, N, profs, 0.5, pid=pid)
    assert_same(g, o)


def test_one_fma_key_falls_back_to_exact_key():
    """The headline's one-fma key holds for values in [FLT_MIN, c_lim] (DESIGN
    §6.2); chunks holding a zero, a subnormal or a value above c_lim (here
    1e5-1e7 spikes, far above 85 y_min Kc / |w_lag|) are redone with the exact
    key.  Choices, totals and statuses must still equal the oracle's."""
    rng = np.random.default_rng(21)
    n, N = 96, 24 + 5000
    tr = inputs.synth_traces_host(n, N, seed=33)
    for i in range(0, n, 3):
        w = rng.integers(24, N, 6)
        tr[i, w[:2]] = 0.0                                   # zeros (valid)
        tr[i, w[2]] = np.float32(1e-40)                      # a subnormal (valid)
        tr[i, w[3:]] = np.float32(rng.choice([1e5, 3e6, 1e7]))  # spikes above c_lim
    tr[5, 3000] = -1.0                                       # invalid (status 4) inside a redone chunk
    J = np.full(n, 3600.0 * (N - 24) * float(RESNET.throughput_sps.min()))
    for eta in (0.5, 0.8):
        g = gpu_plan(tr, N, [RESNET], eta, J=J)
        o = oracle_plan(tr, N, [RESNET], eta, J=J)
        assert o["totals"]["status"][5] == 4
        assert_same(g, o, exact=False)   # the subnormal's products make the sum order visible
