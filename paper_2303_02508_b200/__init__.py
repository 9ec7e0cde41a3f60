"""B200-native batched trace-replay planner for Chase (arXiv 2303.02508).

Thin ctypes binding of libchase.so (include/chase.h): argument marshalling
only — every step of the planner (fit, predict, Eq. 6 argmin, replay, sums)
runs in the library's sm_100a kernels.  PyTorch provides device memory,
streams and process groups.  There is no CPU fallback: importing this package
without the built library raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CHASE_LIB_OVERRIDE") or os.path.join(_HERE, "libchase.so")  # override: A/B builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python build.py` (no CPU fallback exists)")

_lib = ctypes.CDLL(LIB_PATH)

i32, i64, f64, vp, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t

CHASE_F32, CHASE_F64 = 0, 1
STATUS = {0: "OK", 2: "INVALID", 3: "TRACE_EXHAUSTED", 4: "DATA", 5: "MAXCI", 6: "FIT", 7: "CHOICE", 8: "ZERO_ACTUAL",
          10: "CUDA", 11: "NCCL", 12: "WORKSPACE"}


class Traces(ctypes.Structure):
    _fields_ = [("data", vp), ("dtype", i32), ("interval_s", i32), ("n_traces", i64), ("n_steps", i64),
                ("ld", i64), ("phase0", i32), ("reserved", i32)]


class ForecastCfg(ctypes.Structure):
    _fields_ = [("steps_per_day", i32), ("history_len", i32), ("refit_stride", i32), ("period_steps", i32),
                ("ridge_lambda", f64), ("singular_tol", f64), ("forecaster", i32), ("svr_max_iter", i32),
                ("svr_C", f64), ("svr_eps", f64), ("svr_gamma", f64), ("svr_tol", f64)]


FC_LINEAR, FC_SVR = 0, 1
SVR_DEFAULTS = dict(C=1.0, eps=0.1, gamma=0.0, tol=1e-3, max_iter=10000)


class Profile(ctypes.Structure):
    _fields_ = [("n_limits", i32), ("reserved", i32), ("limit_w", ctypes.POINTER(i32)),
                ("avg_power_w", ctypes.POINTER(f64)), ("throughput_sps", ctypes.POINTER(f64))]


class CostCfg(ctypes.Structure):
    _fields_ = [("eta", ctypes.POINTER(f64)), ("n_eta", i32), ("reserved", i32), ("max_power_w", f64),
                ("max_ci", f64)]


class Diag(ctypes.Structure):
    _fields_ = [("first_bad_trace", i64), ("first_bad_status", i32), ("reserved", i32), ("n_bad", ctypes.c_uint64),
                ("n_exhausted", ctypes.c_uint64), ("n_slow_windows", ctypes.c_uint64),
                ("kernel_path", ctypes.c_uint64), ("n_seq_periods", ctypes.c_uint64), ("reserved2", ctypes.c_uint64)]


# chase_diag_t.kernel_path bits (include/chase.h CHASE_PATH_*)
PATH_HEADLINE, PATH_H_PERIODS, PATH_GENERAL, PATH_FC_IN, PATH_ROLL_FUSED = 1, 2, 4, 8, 16


TOTALS_DTYPE = np.dtype([("time_s", "f8"), ("energy_j", "f8"), ("carbon_g", "f8"), ("samples", "f8"),
                         ("base_time_s", "f8"), ("base_energy_j", "f8"), ("base_carbon_g", "f8"),
                         ("completion_window", "i4"), ("status", "i4")])
SUM_FIELDS = ("time_s", "energy_j", "carbon_g", "samples", "base_time_s", "base_energy_j", "base_carbon_g", "n_ok")

_P = ctypes.POINTER
_lib.chase_workspace_bytes.argtypes = [_P(Traces), _P(ForecastCfg), i32, i32]
_lib.chase_workspace_bytes.restype = sz
_lib.chase_fit_forecast.argtypes = [_P(Traces), _P(ForecastCfg), vp, i64, vp, vp, vp, sz, vp]
_lib.chase_fit_forecast.restype = ctypes.c_int
_lib.chase_plan_power_limits.argtypes = [vp, i64, i64, i64, _P(Profile), i32, vp, _P(CostCfg), vp, vp, i64, vp, sz, vp]
_lib.chase_plan_power_limits.restype = ctypes.c_int
_lib.chase_replay.argtypes = [_P(Traces), i32, vp, i64, i32, _P(Profile), i32, vp, vp, vp, vp, vp, sz, vp]
_lib.chase_replay.restype = ctypes.c_int
_lib.chase_sweep.argtypes = [_P(Traces), _P(ForecastCfg), _P(Profile), i32, vp, _P(CostCfg), vp, vp, i64, vp, i64,
                             vp, vp, vp, vp, sz, vp]
_lib.chase_sweep.restype = ctypes.c_int
_lib.chase_forecast_mape.argtypes = [_P(Traces), _P(ForecastCfg), vp, vp, vp, sz, vp]
_lib.chase_forecast_mape.restype = ctypes.c_int
_lib.chase_timeline.argtypes = [_P(Traces), i32, i32, vp, i64, vp, i64, _P(Profile), i32, vp, vp, vp, i64, vp, vp,
                                vp, sz, vp]
_lib.chase_timeline.restype = ctypes.c_int
_lib.chase_period_costs.argtypes = [vp, i64, i64, i64, i32, _P(Profile), i32, vp, _P(CostCfg), vp, vp, i64, vp, i32,
                                    vp, sz, vp]
_lib.chase_period_costs.restype = ctypes.c_int
_lib.chase_profiling_overhead.argtypes = [_P(Traces), i32, _P(Profile), i32, vp, vp, vp, sz, vp]
_lib.chase_profiling_overhead.restype = ctypes.c_int
_lib.chase_diag_read.argtypes = [vp, _P(Diag), vp]
_lib.chase_diag_read.restype = ctypes.c_int
_lib.chase_sweep_host_staging_bytes.argtypes = [_P(Traces), i64, i32]
_lib.chase_sweep_host_staging_bytes.restype = sz
_lib.chase_sweep_host.argtypes = [_P(Traces), _P(ForecastCfg), _P(Profile), i32, vp, _P(CostCfg), vp, i64, vp, vp, sz,
                                  vp, sz, vp]
_lib.chase_sweep_host.restype = ctypes.c_int
_lib.chase_kernel_launches.restype = ctypes.c_uint64
_lib.chase_set_kernel_events.argtypes = [vp, vp]
_lib.chase_set_kernel_events.restype = None
_lib.chase_last_error.restype = ctypes.c_char_p
_lib.chase_version.restype = ctypes.c_char_p

EXPORTED = ("chase_workspace_bytes", "chase_fit_forecast", "chase_plan_power_limits", "chase_replay",
            "chase_sweep", "chase_sweep_host", "chase_sweep_host_staging_bytes", "chase_forecast_mape", "chase_timeline",
            "chase_period_costs", "chase_profiling_overhead",
            "chase_kernel_launches",
            "chase_set_kernel_events", "chase_diag_read", "chase_last_error", "chase_version")


class ChaseError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = _lib.chase_last_error().decode()
        super().__init__(f"{where}: CHASE_ERR_{STATUS.get(code, code)} ({code}): {msg}")


def _check(rc: int, where: str):
    if rc != 0:
        raise ChaseError(rc, where)


def version() -> str:
    return _lib.chase_version().decode()


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


# ------------------------------------------------------------------ marshalling helpers
def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return ctypes.c_void_p(getattr(stream, "cuda_stream", stream))


def make_traces(x, *, n_steps: int | None = None, interval_s: int = 3600, phase0: int = 0) -> Traces:
    """Describe a [n_traces][ld] float32/float64 tensor (device or host memory)."""
    import torch
    assert x.dim() == 2 and x.is_contiguous()
    dt = {torch.float32: CHASE_F32, torch.float64: CHASE_F64}[x.dtype]
    return Traces(x.data_ptr(), dt, interval_s, x.shape[0], n_steps or x.shape[1], x.shape[1], phase0, 0)


def make_fcfg(*, interval_s: int = 3600, history_len: int = 24, refit_stride: int = 0, period_steps: int = 0,
              ridge: float = 1e-8, tol: float = 1e-12, svr=None) -> ForecastCfg:
    """svr: None for the Eq. 1 least-squares forecaster, else a dict of SVR
    hyperparameters (keys of SVR_DEFAULTS; {} = the defaults)."""
    if svr is None:
        return ForecastCfg(86400 // interval_s, history_len, refit_stride, period_steps, ridge, tol, FC_LINEAR, 0,
                           0.0, 0.0, 0.0, 0.0)
    h = dict(SVR_DEFAULTS)
    h.update(svr)
    return ForecastCfg(86400 // interval_s, history_len, refit_stride, period_steps, ridge, tol, FC_SVR,
                       int(h["max_iter"]), float(h["C"]), float(h["eps"]), float(h["gamma"]), float(h["tol"]))


class _Profiles:
    """Keeps the host arrays of a profile list alive for the call."""

    def __init__(self, profiles):
        self.keep = []
        arr = (Profile * len(profiles))()
        for q, p in enumerate(profiles):
            lim = np.ascontiguousarray(p.limit_w, dtype=np.int32)
            pw = np.ascontiguousarray(p.avg_power_w, dtype=np.float64)
            th = np.ascontiguousarray(p.throughput_sps, dtype=np.float64)
            self.keep += [lim, pw, th]
            arr[q] = Profile(len(lim), 0, lim.ctypes.data_as(_P(i32)), pw.ctypes.data_as(_P(f64)),
                             th.ctypes.data_as(_P(f64)))
        self.arr = arr
        self.n = len(profiles)


class _Cost:
    def __init__(self, etas, max_power_w=0.0, max_ci=0.0):
        self.eta = np.ascontiguousarray(etas, dtype=np.float64)
        self.cfg = CostCfg(self.eta.ctypes.data_as(_P(f64)), len(self.eta), 0, float(max_power_w), float(max_ci))


def workspace_bytes(traces: Traces, fcfg: ForecastCfg | None, n_profiles: int, n_eta: int) -> int:
    return int(_lib.chase_workspace_bytes(ctypes.byref(traces), ctypes.byref(fcfg) if fcfg else None,
                                          n_profiles, n_eta))


def alloc_workspace(nbytes: int, device):
    import torch
    # torch allocations are 256-byte aligned (512 in practice)
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)


# ------------------------------------------------------------------ the four entry points
def fit_forecast(traces: Traces, fcfg: ForecastCfg, forecast, ld_f: int, workspace, *, max_ci=None,
                 models=None, stream=None):
    _check(_lib.chase_fit_forecast(ctypes.byref(traces), ctypes.byref(fcfg), _ptr(forecast), ld_f, _ptr(max_ci),
                                   _ptr(models), _ptr(workspace), workspace.numel(), _stream(stream)),
           "chase_fit_forecast")


def plan_power_limits(forecast, n_traces: int, W: int, ld_f: int, profiles, etas, choice, ld_c: int, workspace, *,
                      profile_id=None, max_power_w=0.0, max_ci=0.0, max_ci_per_trace=None, stream=None):
    P, C = _Profiles(profiles), _Cost(etas, max_power_w, max_ci)
    _check(_lib.chase_plan_power_limits(_ptr(forecast), n_traces, W, ld_f, P.arr, P.n, _ptr(profile_id),
                                        ctypes.byref(C.cfg), _ptr(max_ci_per_trace), _ptr(choice), ld_c,
                                        _ptr(workspace), workspace.numel(), _stream(stream)),
           "chase_plan_power_limits")


def replay(traces: Traces, history_len: int, choice, ld_c: int, n_eta: int, profiles, workspace, out_sum, *,
           profile_id=None, job_samples=None, per_trace=None, stream=None):
    P = _Profiles(profiles)
    _check(_lib.chase_replay(ctypes.byref(traces), history_len, _ptr(choice), ld_c, n_eta, P.arr, P.n,
                             _ptr(profile_id), _ptr(job_samples), _ptr(per_trace), _ptr(out_sum),
                             _ptr(workspace), workspace.numel(), _stream(stream)), "chase_replay")


def sweep(traces: Traces, fcfg: ForecastCfg, profiles, etas, workspace, out_sum, *, profile_id=None,
          job_samples=None, choice=None, ld_c: int = 0, forecast=None, ld_f: int = 0, per_trace=None,
          max_power_w=0.0, max_ci=0.0, stream=None):
    P, C = _Profiles(profiles), _Cost(etas, max_power_w, max_ci)
    _check(_lib.chase_sweep(ctypes.byref(traces), ctypes.byref(fcfg), P.arr, P.n, _ptr(profile_id),
                            ctypes.byref(C.cfg), _ptr(job_samples), _ptr(choice), ld_c, _ptr(forecast), ld_f,
                            _ptr(per_trace), _ptr(out_sum), None, _ptr(workspace), workspace.numel(),
                            _stream(stream)), "chase_sweep")


def forecast_mape(traces: Traces, fcfg: ForecastCfg, mape, workspace, *, status=None, stream=None):
    """chase_forecast_mape: walk-forward MAPE of the fit-once model and of
    persistence per trace (mape: f64 [n][2] device tensor; status: int32 [n])."""
    _check(_lib.chase_forecast_mape(ctypes.byref(traces), ctypes.byref(fcfg), _ptr(mape), _ptr(status),
                                    _ptr(workspace), workspace.numel(), _stream(stream)), "chase_forecast_mape")


def timeline(traces: Traces, history_len: int, profiles, rows, m: int, workspace, *, period_steps=1, choice=None,
             ld_c: int = 0, forecast=None, ld_f: int = 0, profile_id=None, job_samples=None, trace_ids=None,
             summary=None, stream=None):
    """chase_timeline: per-period audit rows [m][ceil(W/P)][8] of a planned replay
    (choice None: the max-limit baseline); summary [m][4]: stepwise and Eq. 3
    carbon, AvgPower, AvgCI over the job's run."""
    Pr = _Profiles(profiles)
    _check(_lib.chase_timeline(ctypes.byref(traces), history_len, period_steps, _ptr(choice), ld_c, _ptr(forecast),
                               ld_f, Pr.arr, Pr.n, _ptr(profile_id), _ptr(job_samples), _ptr(trace_ids), m,
                               _ptr(rows), _ptr(summary), _ptr(workspace), workspace.numel(), _stream(stream)),
           "chase_timeline")


def profiling_overhead(traces: Traces, history_len: int, profiles, out, workspace, *, profile_id=None, stream=None):
    """chase_profiling_overhead: [n][3] {time s, energy J, carbon g} of profiling the K limits before the job."""
    P = _Profiles(profiles)
    _check(_lib.chase_profiling_overhead(ctypes.byref(traces), history_len, P.arr, P.n, _ptr(profile_id), _ptr(out),
                                         _ptr(workspace), workspace.numel(), _stream(stream)),
           "chase_profiling_overhead")


def period_costs(forecast, n_traces: int, W: int, ld_f: int, profiles, eta: float, costs, ld_k: int, m: int,
                 workspace, *, period_steps=1, profile_id=None, max_power_w=0.0, max_ci=0.0, max_ci_per_trace=None,
                 trace_ids=None, stream=None):
    """chase_period_costs: Eq. 6 cost vectors [m][ceil(W/P)][ld_k] behind each decision."""
    P, C = _Profiles(profiles), _Cost([eta], max_power_w, max_ci)
    _check(_lib.chase_period_costs(_ptr(forecast), n_traces, W, ld_f, period_steps, P.arr, P.n, _ptr(profile_id),
                                   ctypes.byref(C.cfg), _ptr(max_ci_per_trace), _ptr(trace_ids), m, _ptr(costs), ld_k,
                                   _ptr(workspace), workspace.numel(), _stream(stream)), "chase_period_costs")


def kernel_launches() -> int:
    """Kernels this thread launched through libchase so far."""
    return int(_lib.chase_kernel_launches())


def set_kernel_events(start=None, stop=None):
    """Record torch.cuda.Event `start`/`stop` around the dominant kernel of the
    next calls (None clears).  The events must already exist on the device
    (record them once before passing)."""
    if start is None or stop is None:
        _lib.chase_set_kernel_events(None, None)
    else:
        _lib.chase_set_kernel_events(ctypes.c_void_p(start.cuda_event), ctypes.c_void_p(stop.cuda_event))


def sweep_host_staging_bytes(traces: Traces, chunk_traces: int, n_eta: int) -> int:
    return int(_lib.chase_sweep_host_staging_bytes(ctypes.byref(traces), chunk_traces, n_eta))


def sweep_host(h_traces: Traces, fcfg: ForecastCfg, profiles, etas, chunk_traces: int, staging, workspace, *,
               h_profile_id=None, h_job_samples=None, max_power_w=0.0, max_ci=0.0, stream=None) -> np.ndarray:
    """chase_sweep_host: traces / profile ids / job budgets in HOST memory
    (numpy arrays or pinned torch tensors); returns the host sums [n_eta][8]."""
    P, C = _Profiles(profiles), _Cost(etas, max_power_w, max_ci)
    out = np.zeros((len(C.eta), 8), dtype=np.float64)

    def hp(a):
        if a is None:
            return None
        return ctypes.c_void_p(a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data)

    _check(_lib.chase_sweep_host(ctypes.byref(h_traces), ctypes.byref(fcfg), P.arr, P.n, hp(h_profile_id),
                                 ctypes.byref(C.cfg), hp(h_job_samples), chunk_traces, out.ctypes.data,
                                 _ptr(staging), staging.numel(), _ptr(workspace), workspace.numel(),
                                 _stream(stream)), "chase_sweep_host")
    return out


def diag_read(workspace, stream=None) -> Diag:
    d = Diag()
    _check(_lib.chase_diag_read(_ptr(workspace), ctypes.byref(d), _stream(stream)), "chase_diag_read")
    return d


# ------------------------------------------------------------------ convenience planner
@dataclass
class SweepResult:
    sums: "object"          # torch f64 [n_eta][8]
    per_trace: "object"     # torch u8 view of chase_totals_t [n_eta][n][64] or None
    choice: "object"        # torch u8 [n_eta][n][ld_c] or None
    forecast: "object"      # torch f64 [n][ld_f] or None

    def per_trace_numpy(self) -> np.ndarray:
        return self.per_trace.cpu().numpy().view(TOTALS_DTYPE).reshape(self.per_trace.shape[:2])


class Planner:
    """Owns the device workspace and output buffers for repeated sweeps of one
    shape (the bench's hot loop calls `run()` only)."""

    def __init__(self, traces_tensor, *, n_steps: int, profiles, etas, interval_s=3600, history_len=24,
                 phase0=0, profile_id=None, job_samples=None, want_choice=True, want_forecast=False,
                 want_per_trace=False, max_power_w=0.0, max_ci=0.0, refit_stride=0, period_steps=0, svr=None):
        import torch
        self.x = traces_tensor
        dev = traces_tensor.device
        self.tr = make_traces(traces_tensor, n_steps=n_steps, interval_s=interval_s, phase0=phase0)
        self.fcfg = make_fcfg(interval_s=interval_s, history_len=history_len, refit_stride=refit_stride,
                              period_steps=period_steps, svr=svr)
        self.profiles, self.etas = profiles, list(etas)
        n, W = traces_tensor.shape[0], n_steps - history_len
        self.n, self.W = n, W
        self.ld_c = round_up(W, 16)
        self.ld_f = round_up(W, 2)
        self.ws = alloc_workspace(workspace_bytes(self.tr, self.fcfg, len(profiles), len(self.etas)), dev)
        self.sums = torch.zeros((len(self.etas), 8), dtype=torch.float64, device=dev)
        self.choice = torch.empty((len(self.etas), n, self.ld_c), dtype=torch.uint8, device=dev) if want_choice else None
        self.forecast = torch.empty((n, self.ld_f), dtype=torch.float64, device=dev) if want_forecast else None
        self.per_trace = (torch.empty((len(self.etas), n, 64), dtype=torch.uint8, device=dev)
                          if want_per_trace else None)
        self.profile_id, self.job = profile_id, job_samples
        self.max_power_w, self.max_ci = max_power_w, max_ci
        self._P = _Profiles(profiles)
        self._C = _Cost(self.etas, max_power_w, max_ci)

    def run(self, stream=None):
        _check(_lib.chase_sweep(ctypes.byref(self.tr), ctypes.byref(self.fcfg), self._P.arr, self._P.n,
                                _ptr(self.profile_id), ctypes.byref(self._C.cfg), _ptr(self.job), _ptr(self.choice),
                                self.ld_c, _ptr(self.forecast), self.ld_f, _ptr(self.per_trace), _ptr(self.sums),
                                None, _ptr(self.ws), self.ws.numel(), _stream(stream)), "chase_sweep")
        return SweepResult(self.sums, self.per_trace, self.choice, self.forecast)

    def diag(self) -> Diag:
        return diag_read(self.ws)
