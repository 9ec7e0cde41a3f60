"""Seeded synthetic inputs shared by the oracle tests and the product harness.

Holds none of the planner's arithmetic: only the counter-based
trace generator (C / CUDA in chase_gen.h, bit-identical on host and device),
the synthetic power/throughput profile tables, and the named workload presets
of BASELINE.json configs[0..4].
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libchasegen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python build.py` first")
        lib = ctypes.CDLL(path)
        i64, u64, i32, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p
        lib.chasegen_fill_host.argtypes = [vp, i64, i64, i64, u64, i64, i32, i32, i32, vp, vp]
        lib.chasegen_fill_host.restype = None
        lib.chasegen_profile_ids_host.argtypes = [vp, i64, u64, i64, i32]
        lib.chasegen_profile_ids_host.restype = None
        lib.chasegen_fill_device.argtypes = [vp, i64, i64, i64, u64, i64, i32, i32, i32, vp, vp, vp]
        lib.chasegen_fill_device.restype = ctypes.c_int
        lib.chasegen_profile_ids_device.argtypes = [vp, i64, u64, i64, i32, vp]
        lib.chasegen_profile_ids_device.restype = ctypes.c_int
        _LIB = lib
    return _LIB


MODE_RANDOM, MODE_PAPER = 0, 1


def sin_q_table(T: int) -> np.ndarray:
    """round(2^30 sin(2 pi phi / T)) — the generator's diurnal shape."""
    return np.array([round(math.sin(2.0 * math.pi * p / T) * (1 << 30)) for p in range(T)], dtype=np.int32)


def year_q_table() -> np.ndarray:
    """round(2^30 cos(2 pi d / 365)) — the generator's seasonal shape."""
    return np.array([round(math.cos(2.0 * math.pi * d / 365) * (1 << 30)) for d in range(365)], dtype=np.int32)


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def synth_traces_host(n: int, N: int, *, seed: int, mode: int = MODE_RANDOM, T: int = 24,
                      phase0: int = 0, trace0: int = 0, ld: int | None = None) -> np.ndarray:
    """fp32 [n][ld] traces (g/kWh, multiples of 1/64) on the host."""
    ld = ld or round_up(N, 4)
    out = np.empty((n, ld), dtype=np.float32)
    sq, yq = sin_q_table(T), year_q_table()
    _lib().chasegen_fill_host(out.ctypes.data, n, N, ld, seed, trace0, mode, T, phase0,
                              sq.ctypes.data, yq.ctypes.data)
    return out


def synth_traces_device(out, N: int, *, seed: int, mode: int = MODE_RANDOM, T: int = 24,
                        phase0: int = 0, trace0: int = 0, stream=None) -> None:
    """Fill a CUDA float32 tensor [n][ld] in place (same values as the host)."""
    import torch
    n, ld = out.shape
    sq = torch.from_numpy(sin_q_table(T)).to(out.device)
    yq = torch.from_numpy(year_q_table()).to(out.device)
    s = stream if stream is not None else torch.cuda.current_stream(out.device).cuda_stream
    rc = _lib().chasegen_fill_device(out.data_ptr(), n, N, ld, seed, trace0, mode, T, phase0,
                                     sq.data_ptr(), yq.data_ptr(), s)
    if rc != 0:
        raise RuntimeError(f"chasegen_fill_device failed: cudaError {rc}")
    torch.cuda.current_stream(out.device).synchronize()


def profile_ids_host(n: int, *, seed: int, n_profiles: int, trace0: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.uint8)
    _lib().chasegen_profile_ids_host(out.ctypes.data, n, seed, trace0, n_profiles)
    return out


def profile_ids_device(out, *, seed: int, n_profiles: int, trace0: int = 0) -> None:
    import torch
    rc = _lib().chasegen_profile_ids_device(out.data_ptr(), out.numel(), seed, trace0, n_profiles,
                                            torch.cuda.current_stream(out.device).cuda_stream)
    if rc != 0:
        raise RuntimeError(f"chasegen_profile_ids_device failed: cudaError {rc}")


# ---------------------------------------------------------------- profiles
# Throughput(p) = thr_max*(1 - exp(-min(p, p_sat)/tau)) (S:251 curve form),
# AvgPower(p) = min(0.97 p, P_draw), p_sat = P_draw/0.97, both rounded to 1/64.
# Shapes are synthetic stand-ins (the A40 curves are not in the paper).
SHAPES = {
    "resnet50": (850.0, 120.0, 290.0),
    "bert": (420.0, 80.0, 260.0),   # saturates: identical 275 W / 300 W rows (tie case)
    "vit": (610.0, 105.0, 280.0),
}


@dataclass
class Profile:
    name: str
    limit_w: np.ndarray       # int32, strictly increasing
    avg_power_w: np.ndarray   # f64
    throughput_sps: np.ndarray  # f64

    @property
    def K(self) -> int:
        return len(self.limit_w)


def make_profile(shape: str, limits) -> Profile:
    thr_max, tau, pdraw = SHAPES[shape]
    psat = pdraw / 0.97
    lim = np.asarray(limits, dtype=np.int32)
    thr = np.array([round(64.0 * thr_max * (1.0 - math.exp(-min(p, psat) / tau))) / 64.0 for p in lim])
    pw = np.array([round(64.0 * min(0.97 * p, pdraw)) / 64.0 for p in lim])
    return Profile(shape, lim, pw, thr)


LIMITS_7 = list(range(150, 301, 25))   # C1: 150..300 W
LIMITS_9 = list(range(100, 301, 25))   # S:270 default set


@dataclass
class Workload:
    """One BASELINE.json config."""
    name: str
    n_traces: int
    n_steps: int
    seed: int
    mode: int
    profiles: list
    etas: list
    interval_s: int = 3600
    history_len: int = 24
    phase0: int = 0
    n_profile_shapes: int = 1
    description: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def T(self) -> int:
        return 86400 // self.interval_s

    @property
    def W(self) -> int:
        return self.n_steps - self.history_len

    @property
    def ld(self) -> int:
        return round_up(self.n_steps, 4)

    def job_samples(self, profile_id: np.ndarray | None = None) -> np.ndarray:
        """J_i = Delta * W * min_k Thr_k (always completes; DESIGN Q13)."""
        per_prof = np.array([self.interval_s * self.W * float(p.throughput_sps.min()) for p in self.profiles])
        if profile_id is None:
            return np.full(self.n_traces, per_prof[0])
        return per_prof[profile_id.astype(np.int64)]


def workload(name: str, n_traces: int | None = None) -> Workload:
    rn = make_profile("resnet50", LIMITS_9)
    if name == "C1":
        w = Workload("C1", 1, 24 + 168, 0, MODE_PAPER, [make_profile("resnet50", LIMITS_7)], [0.5],
                     description="1 synthetic region, 7 days hourly, 7 limits ResNet-50 profile, eta=0.5")
    elif name == "C2":
        w = Workload("C2", 1, 24 + 8760, 0, MODE_PAPER, [rn], [0.5],
                     description="1 region, 1 year hourly, 24-hour lag forecaster, 25 W steps")
    elif name == "C3":
        w = Workload("C3", 64, 24 + 43800, 3, MODE_RANDOM, [rn], [round(0.1 * i, 10) for i in range(11)],
                     description="64 regions x 5 years hourly, eta sweep 0..1 in 11 steps")
    elif name == "C4":
        w = Workload("C4", 100_000, 24 + 8760, 4, MODE_RANDOM,
                     [rn, make_profile("bert", LIMITS_9), make_profile("vit", LIMITS_9)], [0.5],
                     n_profile_shapes=3,
                     description="1e5 traces x 1 year, per-trace ResNet-50/BERT/ViT-shaped tables")
    elif name == "C5":
        w = Workload("C5", 1_000_000, 24 + 8760, 5, MODE_RANDOM, [rn], [0.5],
                     description="1e6 traces x 1 year sharded across the GPUs, NCCL all-reduce of totals")
    else:
        raise KeyError(name)
    if n_traces is not None:
        w.n_traces = n_traces
    return w
