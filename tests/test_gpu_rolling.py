"""The rolling refit fused into the sweep (roll_fused_kernel, DESIGN §6.4;
SURVEY §8(a) a3 and the tolerance contract of §8(c)): sliding raw moments and
a closed-form solve instead of oracle_fit's two-pass sequence per origin.

Bars: choices bit-exact except certified near-ties (the oracle's two lowest
Eq. 6 costs within 1e-9 relative at its forecast: the fused forecast is within
~1e-13 of it); per-trace totals of traces whose choices agree within 1e-9;
statuses exact.  Every test asserts through chase_diag_t.kernel_path that the
fused kernel ran (no forecast output, one eta, fp32, aligned L)."""
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
FIELDS = ("time_s", "energy_j", "carbon_g", "samples", "base_time_s", "base_energy_j", "base_carbon_g")


def fused(tr, N, profiles, eta, R, *, pid=None, J=None, L=24, interval_s=3600, phase0=0, max_ci=0.0,
          expect=cb.PATH_ROLL_FUSED):
    x = torch.from_numpy(np.ascontiguousarray(tr)).to(DEV)
    pl = cb.Planner(x, n_steps=N, profiles=profiles, etas=[eta], interval_s=interval_s, history_len=L, phase0=phase0,
                    profile_id=None if pid is None else torch.from_numpy(np.ascontiguousarray(pid, np.uint8)).to(DEV),
                    job_samples=None if J is None else torch.from_numpy(np.ascontiguousarray(J, np.float64)).to(DEV),
                    want_choice=True, want_forecast=False, want_per_trace=True, refit_stride=R, max_ci=max_ci)
    res = pl.run()
    torch.cuda.synchronize()
    d = pl.diag()
    assert d.kernel_path & expect, f"kernel_path={d.kernel_path:#x}"
    return dict(choice=res.choice.cpu().numpy()[0, :, :N - L], totals=res.per_trace_numpy()[0],
                sums=res.sums.cpu().numpy()[0], diag=d)


def check(g, tr, N, profiles, eta, R, *, pid=None, J=None, L=24, interval_s=3600, phase0=0, max_ci=0.0):
    T = 86400 // interval_s
    o = oracle.plan_batch(np.ascontiguousarray(tr, np.float32), N=N, L=L, T=T, phase0=phase0, refit_stride=R,
                          profiles=profiles, profile_id=pid, etas=[eta], max_ci=max_ci, delta=float(interval_s),
                          job_samples=J)
    oc, ot, of = o["choice"][0], o["totals"][0], o["forecast"]
    gt = g["totals"]
    assert np.array_equal(gt["status"], ot["status"]), np.argwhere(gt["status"] != ot["status"])[:5]
    certified = 0
    for i, w in np.argwhere(g["choice"] != oc):
        if ot["status"][i] != 0:
            continue
        p = profiles[0 if pid is None else int(pid[i])]
        mc = max_ci if max_ci > 0 else float(np.max(tr[i, :L]))
        c = sorted(oracle.cost(eta, p.avg_power_w[k], p.throughput_sps[k], float(p.limit_w[-1]), mc, of[i, w])
                   for k in range(p.K))
        assert c[1] - c[0] <= 1e-9 * abs(c[0]), ("uncertified choice mismatch", i, w, of[i, w], c[:2])
        certified += 1
    ok = (gt["status"] == 0) & ~np.any(g["choice"] != oc, axis=1)
    assert np.array_equal(gt["completion_window"][ok], ot["completion_window"][ok])
    for f in FIELDS:
        np.testing.assert_allclose(gt[f][ok], ot[f][ok], rtol=1e-9, atol=0, err_msg=f)
    return certified


@pytest.mark.parametrize("R,L,N,n,interval,phase0", [
    (1, 24, 24 + 3000, 97, 3600, 0),       # every window refits (the C4 bench mode), several chunks
    (1, 24, 24 + 1023, 33, 3600, 5),       # one window short of a chunk, phase offset
    (5, 24, 24 + 2100, 40, 3600, 0),       # slides of 5 rows
    (24, 24, 24 + 2500, 40, 3600, 3),      # direct sums at every (daily) origin
    (33, 24, 24 + 1500, 20, 3600, 0),      # the largest stride the slot's halo covers
    (48, 24, 24 + 1700, 20, 3600, 0),      # origins before the chunk: rows from HBM
    (1, 48, 48 + 1100, 17, 1800, 7),       # half-hourly (T = 48, L = 48)
    (3, 64, 64 + 900, 9, 900, 0),          # 15-minute data, the longest history (L = 64)
])
def test_rolling_fused_matches_oracle(R, L, N, n, interval, phase0):
    T = 86400 // interval
    tr = inputs.synth_traces_host(n, N, seed=400 + R + L, T=T)
    prof = [inputs.make_profile("resnet50", inputs.LIMITS_9)]
    J = np.full(n, interval * (N - L) * prof[0].throughput_sps.min())
    g = fused(tr, N, prof, 0.5, R, J=J, L=L, interval_s=interval, phase0=phase0)
    cert = check(g, tr, N, prof, 0.5, R, J=J, L=L, interval_s=interval, phase0=phase0)
    assert cert <= 2


def test_rolling_fused_multi_profile_and_fixed_maxci():
    w = inputs.workload("C4", n_traces=120)
    N = 24 + 2000
    tr = inputs.synth_traces_host(w.n_traces, N, seed=w.seed)
    pid = inputs.profile_ids_host(w.n_traces, seed=w.seed, n_profiles=3)
    J = np.array([3600.0 * (N - 24) * float(w.profiles[p].throughput_sps.min()) for p in pid])
    for eta, mc in ((0.3, 0.0), (0.7, 650.0), (1.0, 0.0)):
        g = fused(tr, N, w.profiles, eta, 1, pid=pid, J=J, max_ci=mc)
        check(g, tr, N, w.profiles, eta, 1, pid=pid, J=J, max_ci=mc)


def test_rolling_fused_degenerate_windows_take_the_exact_fit():
    """Constant stretches (a constant target: F2; a constant lag column), a
    pure sinusoid (the ridge branch), invalid values (status 4), all through
    the fused kernel's exact fallback (oracle_fit's sequence)."""
    prof = [inputs.make_profile("vit", inputs.LIMITS_9)]
    N, n = 24 + 1500, 10
    tr = inputs.synth_traces_host(n, N, seed=77)
    tr[0, 300:400] = 512.25                      # constant stretch: constant targets and lags
    tr[1, :] = 300.0                             # constant everywhere
    t = np.arange(N)
    tr[2, :] = np.round((500 + 120 * np.sin(2 * np.pi * t / 24)) * 64) / 64   # pure sinusoid
    tr[3, 700] = -2.0                            # a negative value (status 4)
    tr[4, 900] = np.nan                          # NaN (status 4)
    tr[5, 1000:1030] = 0.0                       # zeros (valid)
    J = np.full(n, 3600.0 * 1000 * prof[0].throughput_sps.min())
    g = fused(tr, N, prof, 0.5, 1, J=J)
    check(g, tr, N, prof, 0.5, 1, J=J)
    assert list(g["totals"]["status"][:6]) == [0, 0, 0, 4, 4, 0]
