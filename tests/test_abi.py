"""CPU checks of the C-ABI boundary (no GPU needed): the library loads and
exports every symbol include/*.h declares, host-side validation rejects bad
arguments before anything is enqueued, and the host half of the Eq. 6 fast
path (the exact envelope bucket table) agrees with the oracle's
canonical argmin wherever it claims a decision."""
import ctypes
import glob
import os
import re
from fractions import Fraction as F

import numpy as np
import pytest

import inputs
import oracle
from conftest import ROOT


def _lib():
    import paper_2303_02508_b200 as cb
    return cb


def test_library_exports_every_declared_symbol():
    cb = _lib()
    declared = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        declared |= set(re.findall(r"\b(chase_\w+)\s*\(", src))
    assert {"chase_sweep", "chase_fit_forecast", "chase_plan_power_limits", "chase_replay"} <= declared
    lib = ctypes.CDLL(cb.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(cb.EXPORTED) <= declared
    assert "sm_100a" in cb.version()


def _args(n=4, N=8784, **kw):
    import torch
    x = torch.zeros((n, N), dtype=torch.float32)
    cb = _lib()
    tr = cb.make_traces(x, n_steps=N)
    for k, v in kw.items():
        setattr(tr, k, v)
    return cb, x, tr


def _ws():
    import torch
    return torch.zeros(1 << 20, dtype=torch.uint8)


def test_validation_rejects_bad_arguments_before_enqueueing():
    import torch
    cb, x, tr = _args()
    prof = inputs.make_profile("resnet50", inputs.LIMITS_9)
    fcfg = cb.make_fcfg()
    s = torch.zeros((1, 8), dtype=torch.float64)
    cases = [
        (dict(etas=[1.5]), "eta"),
        (dict(etas=[0.5] * 17), "n_eta"),
        (dict(etas=[0.5], max_power_w=200.0), "max_power_w"),
    ]
    for kw, needle in cases:
        with pytest.raises(cb.ChaseError) as ei:
            cb.sweep(tr, fcfg, [prof], kw.pop("etas"), _ws(), s, stream=0, **kw)
        assert ei.value.code == 2 and needle in str(ei.value)
    bad = inputs.Profile("bad", np.array([100, 100], np.int32), np.array([90.0, 95.0]), np.array([1.0, 2.0]))
    with pytest.raises(cb.ChaseError, match="strictly increasing"):
        cb.sweep(tr, fcfg, [bad], [0.5], _ws(), s, stream=0)
    over = inputs.Profile("over", np.array([100, 200], np.int32), np.array([120.0, 150.0]), np.array([1.0, 2.0]))
    with pytest.raises(cb.ChaseError, match="1.05"):
        cb.sweep(tr, fcfg, [over], [0.5], _ws(), s, stream=0)
    # trace / forecaster configuration
    for field, val, needle in [("interval_s", 7, "86400"), ("ld", 8783, "ld"), ("phase0", 24, "phase0")]:
        cb2, x2, tr2 = _args(**{field: val})
        with pytest.raises(cb.ChaseError, match=needle):
            cb.sweep(tr2, fcfg, [prof], [0.5], _ws(), s, stream=0)
    with pytest.raises(cb.ChaseError, match="history_len"):
        cb.sweep(tr, cb.make_fcfg(history_len=4), [prof], [0.5], _ws(), s, stream=0)
    with pytest.raises(cb.ChaseError, match="workspace"):
        import torch as _t
        cb.sweep(tr, fcfg, [prof], [0.5], _t.zeros(256, dtype=_t.uint8), s, stream=0)


def test_workspace_size_scales_with_traces():
    cb, x, tr = _args(n=10)
    a = cb.workspace_bytes(tr, cb.make_fcfg(), 1, 1)
    tr.n_traces = 1_000_010
    b = cb.workspace_bytes(tr, cb.make_fcfg(), 1, 1)
    assert b - a >= 1_000_000 * 64 and a > 0


def _envelope(P, Th, eta, pmax, maxci, xs):
    cb = _lib()
    lib = ctypes.CDLL(cb.LIB_PATH)
    lib.chase_testing_envelope.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p,
                                           ctypes.c_void_p]
    P = np.ascontiguousarray(P, np.float64)
    Th = np.ascontiguousarray(Th, np.float64)
    xs = np.ascontiguousarray(xs, np.float64)
    out = np.empty(len(xs), np.int32)
    n_iv = lib.chase_testing_envelope(len(P), P.ctypes.data, Th.ctypes.data, eta, pmax, maxci, len(xs),
                                      xs.ctypes.data, out.ctypes.data)
    return out, n_iv


def _crossings(P, Th, eta, pmax, maxci):
    """Exact crossing forecasts of every pair of Eq. 6 cost lines (Fractions)."""
    Kc = F(1 - F(eta)) * F(pmax) * F(maxci)
    out = []
    for j in range(len(P)):
        for k in range(j + 1, len(P)):
            aj, ak = F(eta) * F(P[j]), F(eta) * F(P[k])
            den = aj * F(Th[k]) - ak * F(Th[j])
            if den != 0:
                x = Kc * (F(Th[j]) - F(Th[k])) / den
                if x > 0:
                    out.append(float(x))
    return out


@pytest.mark.parametrize("shape", ["resnet50", "bert", "vit"])
@pytest.mark.parametrize("eta", [0.0, 0.1, 0.5, 0.9, 1.0])
def test_envelope_fast_path_equals_canonical(shape, eta):
    prof = inputs.make_profile(shape, inputs.LIMITS_9)
    P, Th = prof.avg_power_w, prof.throughput_sps
    rng = np.random.default_rng(int(eta * 10) + len(shape))
    for maxci in (750.0, float(rng.uniform(50, 900)), 1.0 / 64):
        xs = list(rng.uniform(0, 3000, 3000)) + [0.0, 1e-300, 5e-324, 1e300]
        for xc in _crossings(P, Th, eta, 300.0, maxci):      # adversarial: +-300 ulps
            x = xc
            for _ in range(300):
                x = np.nextafter(x, -np.inf)
            for _ in range(601):
                xs.append(x)
                x = np.nextafter(x, np.inf)
            xs += [xc * (1 + d) for d in (-1e-6, -1e-9, -1e-12, 1e-12, 1e-9, 1e-6)]
        xs = np.array(xs)
        out, n_iv = _envelope(P, Th, eta, 300.0, maxci, xs)
        assert n_iv >= 1
        fast = out >= 0
        for x, k in zip(xs[fast], out[fast]):
            assert k == oracle.choose(P, Th, eta, 300.0, maxci, x), (x, k)
        # random forecasts almost never need the canonical path
        assert fast[:3000].mean() > 0.999


def test_envelope_random_profiles():
    rng = np.random.default_rng(7)
    for _ in range(150):
        K = int(rng.integers(2, 17))
        lim = np.sort(rng.choice(np.arange(50, 700, 5), K, replace=False)).astype(np.int32)
        Th = np.sort(np.round(rng.uniform(50, 2000, K) * 64) / 64)
        P = np.round(np.minimum(lim * rng.uniform(0.5, 1.04, K), lim * 1.04) * 64) / 64
        if rng.random() < 0.3:
            Th[-1], P[-1] = Th[-2], P[-2]
        eta = float(rng.choice([0.0, 1.0, rng.uniform()]))
        maxci = float(rng.uniform(10, 1500))
        xs = np.concatenate([rng.uniform(0, 4000, 400), np.array(_crossings(P, Th, eta, float(lim[-1]), maxci))])
        out, _ = _envelope(P, Th, eta, float(lim[-1]), maxci, xs)
        for x, k in zip(xs, out):
            if k >= 0:
                assert k == oracle.choose(P, Th, eta, float(lim[-1]), maxci, x)


def test_rolling_workspace_adds_phase_tables_and_forecast_scratch():
    """Rolling refit (refit_stride >= 1) needs the per-phase fit
    tables, and an f64 forecast scratch of round_up(W, 2) per trace only for
    the shapes that do not run in place (here two etas: the exact path and
    the general sweep); one eta on aligned fp32 traces runs the fused kernel
    and writes no forecasts.  Decision periods likewise."""
    cb, x, tr = _args(n=10)
    W = tr.n_steps - 24
    scratch = 10 * ((W + 1) // 2 * 2) * 8
    for f in (cb.make_fcfg(refit_stride=1), cb.make_fcfg(period_steps=24)):
        a1, b1 = cb.workspace_bytes(tr, cb.make_fcfg(), 1, 1), cb.workspace_bytes(tr, f, 1, 1)
        assert b1 - a1 < scratch, (b1 - a1, scratch)
    # (periods with several etas over few traces run as one-eta sweeps: no scratch either)
    f = cb.make_fcfg(refit_stride=1)
    a2, b2 = cb.workspace_bytes(tr, cb.make_fcfg(), 1, 2), cb.workspace_bytes(tr, f, 1, 2)
    assert b2 - a2 >= scratch, (b2 - a2, scratch)
    with pytest.raises(cb.ChaseError, match="refit_stride"):
        prof = inputs.make_profile("resnet50", inputs.LIMITS_9)
        import torch
        cb.sweep(tr, cb.make_fcfg(refit_stride=-1), [prof], [0.5], _ws(), torch.zeros((1, 8), dtype=torch.float64),
                 stream=0)


def test_decision_periods_validation_and_workspace():
    import torch
    cb, x, tr = _args(n=10)
    # one eta on aligned fp32 traces: periods run in the headline kernel, no forecast
    # scratch; fp64 traces take the forecast-first path and need it
    a = cb.workspace_bytes(tr, cb.make_fcfg(), 1, 1)
    b = cb.workspace_bytes(tr, cb.make_fcfg(period_steps=24), 1, 1)
    W = tr.n_steps - 24
    assert b == a
    _, _, tr64 = _args(n=10)
    tr64.dtype = 1  # CHASE_F64
    a = cb.workspace_bytes(tr64, cb.make_fcfg(), 1, 1)
    b = cb.workspace_bytes(tr64, cb.make_fcfg(period_steps=24), 1, 1)
    assert b - a >= 10 * ((W + 1) // 2 * 2) * 8
    prof = inputs.make_profile("resnet50", inputs.LIMITS_9)
    s = torch.zeros((1, 8), dtype=torch.float64)
    for f, needle in [(cb.make_fcfg(period_steps=-1), "period_steps"),
                      (cb.make_fcfg(period_steps=4, refit_stride=2), "refit_stride")]:
        with pytest.raises(cb.ChaseError, match=needle):
            cb.sweep(tr, f, [prof], [0.5], _ws(), s, stream=0)


def test_svr_forecaster_validation_and_workspace():
    """f2: the SVR forecaster adds the per-trace dual models and the forecast
    scratch to the workspace, and rejects what it does not support."""
    import torch
    cb, x, tr = _args(n=10)
    a = cb.workspace_bytes(tr, cb.make_fcfg(), 1, 1)
    b = cb.workspace_bytes(tr, cb.make_fcfg(svr={}), 1, 1)
    W = tr.n_steps - 24
    assert b - a >= 10 * ((W + 1) // 2 * 2) * 8 + 10 * 268 * 8
    f = cb.make_fcfg(svr={})
    assert (f.forecaster, f.svr_C, f.svr_eps, f.svr_gamma, f.svr_tol, f.svr_max_iter) == (1, 1.0, 0.1, 0.0, 1e-3, 10000)
    prof = inputs.make_profile("resnet50", inputs.LIMITS_9)
    s = torch.zeros((1, 8), dtype=torch.float64)
    bad_kind = cb.make_fcfg()
    bad_kind.forecaster = 7
    for f, needle in [(bad_kind, "forecaster"),
                      (cb.make_fcfg(svr={}, refit_stride=24), "refit_stride"),
                      (cb.make_fcfg(svr={}, history_len=65), "history_len"),
                      (cb.make_fcfg(svr={"C": 0.0}), "hyperparameters"),
                      (cb.make_fcfg(svr={"eps": -1.0}), "hyperparameters"),
                      (cb.make_fcfg(svr={"tol": 0.0}), "hyperparameters"),
                      (cb.make_fcfg(svr={"gamma": float("nan")}), "hyperparameters"),
                      (cb.make_fcfg(svr={"max_iter": -1}), "hyperparameters")]:
        with pytest.raises(cb.ChaseError, match=needle):
            cb.sweep(tr, f, [prof], [0.5], _ws(), s, stream=0)
    with pytest.raises(cb.ChaseError, match="d_models"):
        cb.fit_forecast(tr, cb.make_fcfg(svr={}), _ws(), W, _ws(), models=_ws(), stream=0)
