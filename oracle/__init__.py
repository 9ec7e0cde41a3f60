"""ctypes binding of liboracle.so — the plain CPU oracle (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  The product (paper_2303_02508_b200) never does.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

i32, i64, f64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class Model(ctypes.Structure):
    _fields_ = [("c0", f64), ("ws", f64), ("wc", f64), ("wl", f64),
                ("mu", f64 * 4), ("sigma", f64 * 4),
                ("kind", i32), ("ridge", i32), ("status", i32), ("n_cols", i32)]


class Totals(ctypes.Structure):
    _fields_ = [("time_s", f64), ("energy_j", f64), ("carbon_g", f64), ("samples", f64),
                ("base_time_s", f64), ("base_energy_j", f64), ("base_carbon_g", f64),
                ("completion_window", i32), ("status", i32)]


TOTALS_DTYPE = np.dtype([("time_s", "f8"), ("energy_j", "f8"), ("carbon_g", "f8"), ("samples", "f8"),
                         ("base_time_s", "f8"), ("base_energy_j", "f8"), ("base_carbon_g", "f8"),
                         ("completion_window", "i4"), ("status", "i4")])
assert TOTALS_DTYPE.itemsize == ctypes.sizeof(Totals) == 64


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python build.py` first")
        L = ctypes.CDLL(path)
        L.oracle_phase_table.argtypes = [i32, vp, vp]
        L.oracle_fit.argtypes = [vp, i32, i32, i32, vp, vp, f64, f64, ctypes.POINTER(Model)]
        L.oracle_fit.restype = i32
        L.oracle_predict.argtypes = [ctypes.POINTER(Model), f64, f64, f64]
        L.oracle_predict.restype = f64
        L.oracle_cost.argtypes = [f64] * 6
        L.oracle_cost.restype = f64
        L.oracle_choose.argtypes = [i32, vp, vp, f64, f64, f64, f64]
        L.oracle_choose.restype = i32
        L.oracle_cta.argtypes = [f64, f64, f64]
        L.oracle_cta.restype = f64
        L.oracle_total_cost.argtypes = [f64] * 6
        L.oracle_total_cost.restype = f64
        L.oracle_replay.argtypes = [vp, i32, i32, vp, vp, vp, f64, f64, vp, ctypes.POINTER(i32)]
        L.oracle_replay.restype = i32
        L.oracle_plan_trace.argtypes = [vp, i32, i32, i32, i32, i32, i32, vp, f64, f64, vp, vp, i32, vp, vp,
                                        i32, vp, f64, f64, f64, f64, vp, vp, vp]
        L.oracle_plan_trace.restype = i32
        L.oracle_plan_batch_f32.argtypes = [vp, i64, i64, i64, i32, i32, i32, i32, i32, vp, f64, f64, i32,
                                            vp, vp, vp, vp, vp, vp, i32, vp, f64, f64, f64, vp, vp,
                                            vp, vp, vp, i32]
        L.oracle_plan_batch_f32.restype = i32
        L.oracle_timeline.argtypes = [vp, i32, i32, i32, vp, vp, i32, vp, vp, vp, f64, f64, vp]
        L.oracle_timeline.restype = i32
        L.oracle_job_summary.argtypes = [vp, i32, i32, vp, i32, vp, vp, f64, f64, vp]
        L.oracle_job_summary.restype = None
        L.oracle_profiling_overhead.argtypes = [vp, i32, i32, vp, f64, vp]
        L.oracle_profiling_overhead.restype = i32
        L.oracle_rbf_exp.argtypes = [f64]
        L.oracle_rbf_exp.restype = f64
        L.oracle_svr_fit.argtypes = [vp, i32, i32, i32, vp, vp, f64, f64, f64, f64, i32, ctypes.POINTER(SVRModel)]
        L.oracle_svr_fit.restype = i32
        L.oracle_svr_predict.argtypes = [ctypes.POINTER(SVRModel), f64, f64, f64]
        L.oracle_svr_predict.restype = f64
        L.oracle_mape.argtypes = [vp, vp, i64]
        L.oracle_mape.restype = f64
        L.oracle_evaluate.argtypes = [vp, i32, i32, i32, i32, f64, f64, vp, vp, vp, vp]
        L.oracle_evaluate.restype = i32
        L.oracle_evaluate_batch_f32.argtypes = [vp, i64, i64, i64, i32, i32, i32, f64, f64, vp, vp, vp, i32]
        L.oracle_evaluate_batch_f32.restype = i32
        _LIB = L
    return _LIB


class SVRModel(ctypes.Structure):
    """oracle_svr_t (oracle.h): the epsilon-SVR forecaster (f2)."""
    _fields_ = [("z", (ctypes.c_double * 3) * 63), ("coef", ctypes.c_double * 63), ("mu", ctypes.c_double * 4),
                ("sigma", ctypes.c_double * 4), ("gamma", ctypes.c_double), ("rho", ctypes.c_double),
                ("n", ctypes.c_int32), ("kind", ctypes.c_int32), ("iters", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("keep", ctypes.c_int32 * 3), ("status", ctypes.c_int32)]


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def phase_table(T: int):
    S, C = np.empty(T), np.empty(T)
    lib().oracle_phase_table(T, S.ctypes.data, C.ctypes.data)
    return S, C


def fit(hist, T: int, phi0: int = 0, ridge: float = 1e-8, tol: float = 1e-12) -> Model:
    h = _f64(hist)
    S, C = phase_table(T)
    m = Model()
    lib().oracle_fit(h.ctypes.data, len(h), T, phi0, S.ctypes.data, C.ctypes.data, ridge, tol, ctypes.byref(m))
    return m


def predict(m: Model, s: float, c: float, lag: float) -> float:
    return lib().oracle_predict(ctypes.byref(m), s, c, lag)


def cost(eta, avg_power, thr, pmax, maxci, chat) -> float:
    return lib().oracle_cost(eta, avg_power, thr, pmax, maxci, chat)


def choose(avg_power, thr, eta, pmax, maxci, chat) -> int:
    P, Th = _f64(avg_power), _f64(thr)
    return lib().oracle_choose(len(P), P.ctypes.data, Th.ctypes.data, eta, pmax, maxci, chat)


def cta(tta, p, ci) -> float:
    return lib().oracle_cta(tta, p, ci)


def total_cost(tta, p, ci, eta, pmax, maxci) -> float:
    return lib().oracle_total_cost(tta, p, ci, eta, pmax, maxci)


def replay(c, s0, choice, avg_power, thr, delta, J):
    c = _f64(c)
    ch = np.ascontiguousarray(choice, dtype=np.uint8)
    P, Th = _f64(avg_power), _f64(thr)
    out = np.empty(4)
    w = i32()
    st = lib().oracle_replay(c.ctypes.data, len(c), s0, ch.ctypes.data, P.ctypes.data, Th.ctypes.data,
                             delta, J, out.ctypes.data, ctypes.byref(w))
    return out, w.value, st


def _svr(svr):
    """None (least squares) or a dict of SVR hyperparameters -> the oracle's params array."""
    if svr is None:
        return None
    d = dict(C=1.0, eps=0.1, gamma=0.0, tol=1e-3, max_iter=10000)
    d.update(svr if isinstance(svr, dict) else {})
    return np.array([d["C"], d["eps"], d["gamma"], d["tol"], float(d["max_iter"])], dtype=np.float64)


def plan_trace(c, *, L, T, phase0=0, refit_stride=0, period=1, svr=None, ridge=1e-8, tol=1e-12, avg_power, thr,
               etas, pmax, max_ci=0.0, delta=3600.0, J=0.0):
    c = _f64(c)
    N = len(c)
    W = N - L
    S, C = phase_table(T)
    P, Th, E = _f64(avg_power), _f64(thr), _f64(etas)
    fc = np.empty(W)
    ch = np.empty((len(E), W), dtype=np.uint8)
    tot = np.zeros(len(E), dtype=TOTALS_DTYPE)
    sv = _svr(svr)
    st = lib().oracle_plan_trace(c.ctypes.data, N, L, T, phase0, refit_stride, period,
                                 None if sv is None else sv.ctypes.data, ridge, tol,
                                 S.ctypes.data, C.ctypes.data, len(P), P.ctypes.data, Th.ctypes.data,
                                 len(E), E.ctypes.data, pmax, max_ci, delta, J,
                                 fc.ctypes.data, ch.ctypes.data, tot.ctypes.data)
    return fc, ch, tot, st


def plan_batch(traces, *, N, L, T, phase0=0, refit_stride=0, period=1, svr=None, ridge=1e-8, tol=1e-12, profiles,
               profile_id=None, etas, pmax=0.0, max_ci=0.0, delta=3600.0, job_samples=None,
               want_forecast=True, want_choice=True, threads=0):
    """traces: float32 [n][ld].  profiles: list of objects with limit_w,
    avg_power_w, throughput_sps.  Returns dict(forecast, choice, totals, sums, threads)."""
    tr = np.ascontiguousarray(traces, dtype=np.float32)
    n, ld = tr.shape
    W = N - L
    Ks = np.array([len(p.limit_w) for p in profiles], dtype=np.int32)
    offs = np.concatenate([[0], np.cumsum(Ks)[:-1]]).astype(np.int32)
    P = _f64(np.concatenate([p.avg_power_w for p in profiles]))
    Th = _f64(np.concatenate([p.throughput_sps for p in profiles]))
    pm = _f64([float(max(p.limit_w)) for p in profiles])
    E = _f64(etas)
    sv = _svr(svr)
    pid = None if profile_id is None else np.ascontiguousarray(profile_id, dtype=np.uint8)
    job = None if job_samples is None else _f64(job_samples)
    fc = np.empty((n, W)) if want_forecast else None
    ch = np.empty((len(E), n, W), dtype=np.uint8) if want_choice else None
    tot = np.zeros((len(E), n), dtype=TOTALS_DTYPE)
    sums = np.zeros((len(E), 8))
    used = lib().oracle_plan_batch_f32(
        tr.ctypes.data, n, N, ld, L, T, phase0, refit_stride, period, None if sv is None else sv.ctypes.data,
        ridge, tol, len(profiles),
        Ks.ctypes.data, offs.ctypes.data, P.ctypes.data, Th.ctypes.data, pm.ctypes.data,
        None if pid is None else pid.ctypes.data, len(E), E.ctypes.data, pmax, max_ci, delta,
        None if job is None else job.ctypes.data,
        None if fc is None else fc.ctypes.data, None if ch is None else ch.ctypes.data,
        tot.ctypes.data, sums.ctypes.data, threads)
    return dict(forecast=fc, choice=ch, totals=tot, sums=sums, threads=used)


def mape(actual, predicted) -> float:
    """SPEC mape: 100/n * sum |a - p| / |a|; NaN if undefined."""
    a, p = _f64(actual), _f64(predicted)
    assert len(a) == len(p)
    return float(lib().oracle_mape(a.ctypes.data, p.ctypes.data, len(a)))


def evaluate(c, *, L, T, phase0=0, ridge=1e-8, tol=1e-12, svr=None):
    """SPEC evaluate_models for one trace: (status, mape_linear, mape_persistence)."""
    c = _f64(c)
    S, C = phase_table(T)
    out = np.empty(2)
    sv = _svr(svr)
    st = lib().oracle_evaluate(c.ctypes.data, len(c), L, T, phase0, ridge, tol, S.ctypes.data, C.ctypes.data,
                               None if sv is None else sv.ctypes.data, out.ctypes.data)
    return st, float(out[0]), float(out[1])


def evaluate_batch(traces, *, N, L, T, phase0=0, ridge=1e-8, tol=1e-12, threads=0, svr=None):
    """fp32 traces [n][ld] -> (mape [n][2], status [n], threads used)."""
    tr = np.ascontiguousarray(traces, dtype=np.float32)
    n, ld = tr.shape
    out = np.empty((n, 2))
    st = np.empty(n, dtype=np.int32)
    sv = _svr(svr)
    used = lib().oracle_evaluate_batch_f32(tr.ctypes.data, n, N, ld, L, T, phase0, ridge, tol,
                                           None if sv is None else sv.ctypes.data, out.ctypes.data,
                                           st.ctypes.data, threads)
    return out, st, used


def timeline(c, *, L, period=1, choice=None, forecast=None, limit_w, avg_power, thr, delta=3600.0, J=0.0):
    """SPEC emit_timeline: rows [n_periods][8] = period_start,
    forecast_ci, actual_mean_ci, chosen_limit_w, avg_power_w, samples_done,
    energy_j, carbon_g (choice None: the max-limit baseline)."""
    c = _f64(c)
    N = len(c)
    W = N - L
    P = max(int(period), 1)
    n_per = -(-W // P)
    rows = np.empty((n_per, 8))
    ch = None if choice is None else np.ascontiguousarray(choice, dtype=np.uint8)
    fc = None if forecast is None else _f64(forecast)
    lim = np.ascontiguousarray(limit_w, dtype=np.int32)
    pw, th = _f64(avg_power), _f64(thr)
    n = lib().oracle_timeline(c.ctypes.data, N, L, P, None if ch is None else ch.ctypes.data,
                              None if fc is None else fc.ctypes.data, len(pw), lim.ctypes.data, pw.ctypes.data,
                              th.ctypes.data, delta, J, rows.ctypes.data)
    assert n == n_per
    return rows


def job_summary(c, *, L, choice=None, avg_power, thr, delta=3600.0, J=0.0):
    """Eq. 3 next to the stepwise carbon: [stepwise g, Eq. 3 g, AvgPower W, AvgCI g/kWh]."""
    c = _f64(c)
    ch = None if choice is None else np.ascontiguousarray(choice, dtype=np.uint8)
    pw, th = _f64(avg_power), _f64(thr)
    out = np.empty(4)
    lib().oracle_job_summary(c.ctypes.data, len(c), L, None if ch is None else ch.ctypes.data, len(pw),
                             pw.ctypes.data, th.ctypes.data, delta, J, out.ctypes.data)
    return out


def profiling_overhead(c, *, L, avg_power, delta=3600.0):
    """SPEC --count-profiling: [time s, energy J, carbon g] of profiling the K limits before the job."""
    c = _f64(c)
    pw = _f64(avg_power)
    out = np.empty(3)
    st = lib().oracle_profiling_overhead(c.ctypes.data, L, len(pw), pw.ctypes.data, delta, out.ctypes.data)
    return st, out


def rbf_exp(x: float) -> float:
    return float(lib().oracle_rbf_exp(float(x)))


def svr_fit(hist, *, T, phi0=0, C=1.0, eps=0.1, gamma=0.0, tol=1e-3, max_iter=10000):
    """SPEC fit_svr on the L history points: returns an SVRModel."""
    h = _f64(hist)
    S, Cc = phase_table(T)
    m = SVRModel()
    lib().oracle_svr_fit(h.ctypes.data, len(h), T, phi0, S.ctypes.data, Cc.ctypes.data, C, eps, gamma, tol,
                         max_iter, ctypes.byref(m))
    return m


def svr_predict(m, s, c, lag) -> float:
    return float(lib().oracle_svr_predict(ctypes.byref(m), s, c, lag))
