#!/usr/bin/env python3
"""bench.py — trace-windows planned per second (fit + argmin + replay) on B200.

Metric (BASELINE.json): "trace-windows planned/sec (fit+argmin+replay) at
1/2/4/8 B200; % of HBM peak".  One step = one chase_sweep over this GPU's
batch of traces (fit once, predict, Eq. 6 argmin, fixed-work replay + max-power
baseline, per-GPU totals) plus, for N > 1, the NCCL all-reduce of the totals.

  python bench.py [--gpus N --steps K --warmup W] [--config C5] [--impl reference]

N > 1 is launched by torchrun (one rank per GPU); the workload's traces
(C5: 10^6, configs[4]) are split across the ranks, contiguous and balanced
(strong scaling; --weak gives every rank its own), and rank 0 prints ONE JSON
line.
`--impl reference` times the CPU oracle (oracle/) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402

METRIC = "trace-windows planned/sec (fit+argmin+replay)"
UNIT = "trace-windows/s"
BYTES_PER_WINDOW = 5.0   # 4 B fp32 trace read + 1 B choice write


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["chase", "reference"], default="chase")
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--traces", type=int, default=None,
                    help="override the workload's trace count (total; per GPU with --weak)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank plans its own --traces (default: strong, the workload "
                         "split across the ranks as configs[4] names it)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle time for cpu_baseline")
    ap.add_argument("--e2e-traces", type=int, default=None)
    ap.add_argument("--no-prefix-check", action="store_true",
                    help="skip the untimed oracle parity check of the whole cpu_baseline sample")
    ap.add_argument("--mode", choices=["plan", "mape", "timeline"], default="plan",
                    help="plan: the planner (headline); mape: the walk-forward forecast-evaluation sweep (f3); "
                         "timeline: per-period audit rows of a planned replay (f4)")
    ap.add_argument("--period-steps", type=int, default=0,
                    help="P > 1: one decision per period of P steps on the mean recursive forecast (f1)")
    ap.add_argument("--forecaster", choices=["linear", "svr"], default="linear",
                    help="linear: Eq. 1 least squares (headline); svr: the epsilon-SVR of Table 1 (FP64-bound)")
    ap.add_argument("--refit-stride", type=int, default=0,
                    help="0: fit once at job start (headline); R >= 1: rolling refit every R windows (FP64-bound)")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks
CLOCK_FIELDS = ["timestamp", "index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
                "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
                "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]


class ClockSampler:
    """nvidia-smi clocks and throttle reasons every 20 ms; the samples whose
    timestamps fall in the timed region [begin(), end()] are reported (the one
    nearest the region when it is shorter than the sampling interval)."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None
        self.t_begin = self.t_end = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", "--query-gpu=" + ",".join(CLOCK_FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            t_wait = time.time() + 3.0            # live before the timed region starts
            while time.time() < t_wait and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
            time.sleep(0.05)
        except (OSError, FileNotFoundError):
            self.proc = None

    def begin(self):
        self.t_begin = time.time()

    def end(self):
        self.t_end = time.time()
        time.sleep(0.05)                          # one more sample past the region

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        import datetime
        rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < len(CLOCK_FIELDS):
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[2]), float(parts[3]),
                             {n for n, v in zip(names, parts[6:10]) if v.lower().startswith("active")}))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        b = self.t_begin if self.t_begin is not None else rows[0][0]
        e = self.t_end if self.t_end is not None else rows[-1][0]
        sel = [r for r in rows if b <= r[0] <= e]
        if not sel:                               # a region shorter than the interval: the nearest sample
            mid = 0.5 * (b + e)
            sel = [min(rows, key=lambda r: abs(r[0] - mid))]
        reasons = set().union(*(r[3] for r in sel))
        return {"sm_mhz": float(np.median([r[1] for r in sel])), "sm_max_mhz": float(max(r[2] for r in sel)),
                "reasons": sorted(reasons), "samples": len(sel), "timed_region_s": round(e - b, 4)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic_per_window(config: str):
    """DRAM bytes per planned window of the sweep kernel from the committed
    `ncu --set full` capture summary (profiles/ncu_traffic.json), if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path))
    e = d.get(config) or (None if "_" in config else d.get("default"))
    return None if e is None else float(e["dram_bytes_per_window"])


# ------------------------------------------------------------------ CPU oracle leg
class OracleSample:
    """A bounded prefix sample of the workload, generated once on the host,
    planned by the CPU oracle as it stands (OpenMP across traces)."""

    def __init__(self, w: inputs.Workload, n: int, R: int = 0, P: int = 0, svr=None):
        self.w, self.n, self.R, self.P, self.svr = w, n, R, P, svr
        self.tr = inputs.synth_traces_host(n, w.n_steps, seed=w.seed, mode=w.mode)
        self.pid = (inputs.profile_ids_host(n, seed=w.seed, n_profiles=len(w.profiles))
                    if len(w.profiles) > 1 else None)
        self.J = w.job_samples(self.pid)[:n]
        self.cores = 0

    def run(self) -> float:
        import oracle
        w = self.w
        t0 = time.perf_counter()
        r = oracle.plan_batch(self.tr, N=w.n_steps, L=w.history_len, T=w.T, refit_stride=self.R, period=self.P,
                              svr=self.svr, profiles=w.profiles,
                              profile_id=self.pid, etas=w.etas, delta=float(w.interval_s), job_samples=self.J,
                              want_forecast=False, want_choice=False)
        self.cores = r["threads"]
        return time.perf_counter() - t0


def calibrated_sample(w: inputs.Workload, target_s: float, max_traces: int, R: int = 0, P: int = 0,
                      svr=None) -> OracleSample:
    """Two-stage calibration: a tiny probe (dominated by thread start-up)
    sizes a ~1 s probe, whose rate sizes the sample to ~target_s."""
    n0 = min(max_traces, 256 if R == 0 and svr is None else 4)
    probe = OracleSample(w, n0, R, P, svr)
    dt = probe.run()
    n1 = int(min(max_traces, max(n0, n0 * min(1.0, target_s) / max(dt, 1e-3))))
    if n1 > n0:
        probe = OracleSample(w, n1, R, P, svr)
        dt = probe.run()
        n0 = n1
    n = int(min(max_traces, max(n0, n0 * target_s / max(dt, 1e-3))))
    return probe if n <= n0 else OracleSample(w, n, R, P, svr)


def oracle_sample_rate(w: inputs.Workload, target_s: float, max_traces: int, R: int = 0, P: int = 0, svr=None):
    s = calibrated_sample(w, target_s, max_traces, R, P, svr)
    dt = s.run()
    return s.n * w.W / dt, s.cores, s.n, dt


# ------------------------------------------------------------------ reference arm
def main_reference(args):
    """The CPU oracle, as it stands, on the host cores: same metric/config, each
    step a bounded prefix sample of the workload (rank 0 only under torchrun)."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    w = inputs.workload(args.config, n_traces=args.traces)
    per_step = min(10.0, 150.0 / max(1, args.steps + args.warmup))
    s = calibrated_sample(w, per_step, w.n_traces, args.refit_stride, args.period_steps, svr_arg(args))
    times = []
    for k in range(args.warmup + args.steps):
        dt = s.run()
        if k >= args.warmup:
            times.append(dt)
    step_s = float(np.mean(times))
    value = s.n * w.W / step_s
    sample = (f"first {s.n} of {w.n_traces} traces of {w.name} per step ({s.n * w.W:.3g} windows), "
              f"{s.cores} host threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(w, args.gpus, args.refit_stride, args.period_steps, svr_arg(args),
                                  n_total=w.n_traces * (args.gpus if args.weak else 1), weak=args.weak),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": s.cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def rolling_flops(w: inputs.Workload, R: int) -> float:
    """Algorithmic fp64 operations of one rolling launch: per
    origin the oracle's fit, 42n + 56 for n = L-1 rows (sums 4n, two-pass
    moments 12n, z-scores and Gram/rhs 26n, means/sigmas 8, Cholesky + solves +
    un-standardisation 44, every add/sub/mul/div/sqrt one flop), plus the
    prediction, 6 per window."""
    n = w.history_len - 1
    origins = -(-w.W // R)
    return float(w.n_traces) * (origins * (42 * n + 56) + 6 * w.W)


def rolling_fused_flops(w: inputs.Workload, R: int) -> float:
    """Algorithmic fp64 operations of one roll_fused_kernel launch (DESIGN §6.4,
    the sliding-moment formulation; an fma counts 2, every add/sub/mul/div 1):
    per origin the closed-form solve, 62 (the lag moments 6, seven centred
    moments 21, the two phase-block products 12, s_ll and r_y 8, b_l 1, b_s and
    b_c 4, the means 4, the intercept 6), plus the moments: a slide of R rows at
    32 per row (add one row, remove one: 2 x (1 fma + 2 mul + 6 fma)) when
    R <= 8, else the direct sums of the n = L-1 rows at 16 per row; per window
    the prediction 6, the Eq. 6 key 1 and the replay sums 5."""
    n = w.history_len - 1
    origins = -(-w.W // R)
    mom = 32.0 * R if R <= 8 else 16.0 * n
    return float(w.n_traces) * (origins * (62.0 + mom) + 12.0 * w.W)


def svr_arg(args):
    """The SVR hyperparameters (the binding's defaults: C 1, eps 0.1, gamma 1/3, tol 1e-3) or None."""
    return {} if getattr(args, "forecaster", "linear") == "svr" else None


def svr_flops(w: inputs.Workload) -> float:
    """Algorithmic fp64 operations of the SVR forecaster per launch pair
    (DESIGN §6.8), a LOWER bound, an fma counted as 2: per trace the kernel
    matrix, n^2 RBF entries of 27 flops (squared distance 3 sub + 1 mul + 2 fma
    = 8, gamma 1; exp 18: the nearest-integer shift fma + sub 3, the two
    reduction fma 4, 5 Horner fma 10, the table product 1 -- the 2^e scaling is
    an integer add), plus per window one prediction of 29n + 5 flops (the lag
    z-score 2, n x (RBF 27 + the coef fma 2), bias and un-standardisation 3;
    the sin/cos z-scores are per phase).  The SMO iterations are not counted
    (their number depends on the data)."""
    n = w.history_len - 1
    return float(w.n_traces) * (27.0 * n * n + w.W * (29.0 * n + 5.0))


def fp64_peak():
    """FP64 vector peak in TFLOP/s (a DFMA = 2 flops): the DFMA rate measured
    by tools/fp64_probe.cu (profiles/fp64_probe.json) when present, else
    148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz."""
    path = os.path.join(ROOT, "profiles", "fp64_probe.json")
    if os.path.exists(path):
        for line in open(path):
            d = json.loads(line)
            if d.get("op") == "dfma":
                return 2.0 * d["thread_ops_per_s"] / 1e12, "measured (tools/fp64_probe.cu DFMA rate x 2, profiles/fp64_probe.json)"
    return 148 * 64 * 2 * 1.965e9 / 1e12, "derived (148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz)"


def planner_kernel_name(w: inputs.Workload, R: int = 0, P: int = 0, svr=None) -> str:
    if svr is not None:
        return ("svr_fit_kernel (warp per trace, SMO on the RBF dual, kernel matrix in smem) + "
                "svr_forecast_kernel (thread per window / period)")
    if P > 1:
        if len(w.etas) == 1 and w.history_len % 4 == 0:  # the headline kernel's period instantiations
            if P * 30 >= 1920:
                return ("sweep_fast_kernel<2> (decision periods in 32-period batches, one horizon per lane; "
                        "Eq. 6 argmin + run-form replay)")
            if 60 % P == 0:
                return (f"sweep_fast_kernel<{P + 2 if P in (2, 3, 4, 5, 6, 10, 12, 15) else 3}> (decision periods: each lane decides and replays its own periods; "
                        "Eq. 6 argmin + replay)")
            return ("sweep_fast_kernel<1> (decision periods: per-chunk decisions, up to 4 horizon chains per lane; "
                    "Eq. 6 argmin + replay)")
        return "sweep_kernel<FUSED, FIN> (Eq. 6 argmin + replay on the period decision forecasts)"
    if R > 0:
        if len(w.etas) == 1 and w.history_len % 4 == 0 and w.history_len <= 64:
            return ("roll_fused_kernel (rolling refit fused into the sweep: sliding raw moments + closed-form "
                    "solve per origin, Eq. 6 argmin + replay)")
        return "rolling_forecast_kernel (one thread per (trace, refit origin), oracle_fit's exact fp64 sequence)"
    if len(w.etas) == 1 and w.history_len % 4 == 0:
        return "sweep_fast_kernel (fused predict + Eq. 6 argmin + replay; fp32 traces, one eta)"
    return "sweep_kernel<FUSED> (fused predict + Eq. 6 argmin + replay)"


def workload_config(w: inputs.Workload, n_gpus: int, R: int = 0, P: int = 0, svr=None, n_total=None, weak=False):
    fc = ("fit once per trace on the 24 h before job start (P:67), least squares (Table 1 LR)" if R == 0 else
          f"rolling refit every {R} window(s) on the {w.history_len} points before each origin (P:78-79)")
    if svr is not None:
        fc = ("fit once per trace on the 24 h before job start (P:67), epsilon-SVR with an RBF kernel "
              "(Table 1's best model, P:162; C=1, eps=0.1, gamma=1/3, tol=1e-3)")
    if P > 1:
        fc += f"; one decision per {P}-step period on the mean recursive forecast (P:130, S:158-166)"
    n_total = w.n_traces if n_total is None else n_total
    split = (f"{n_total} traces, {'each of' if weak else 'split across'} {n_gpus} GPU(s) "
             f"({'weak' if weak else 'strong'} scaling)")
    return {
        "workload": f"{w.name}: {w.description}; {split}",
        "traces_total": n_total, "traces_per_gpu": -(-n_total // n_gpus), "steps_per_trace": w.n_steps,
        "history_len": w.history_len,
        "windows_per_trace": w.W, "interval_s": w.interval_s, "n_eta": len(w.etas),
        "n_limits": int(w.profiles[0].K), "profiles": [p.name for p in w.profiles],
        "forecaster": fc, "refit_stride": R, "period_steps": max(P, 1),
        "l2": (f"L2 flushed between timed steps (512 MB write outside each step's CUDA events; "
               f"{n_total * w.ld * 4 / 1e6:.3g} MB of fp32 traces vs the 126 MB L2)" if l2_resident(w, n_total) else
               f"inputs larger than L2 ({n_total * w.ld * 4 / n_gpus / 1e9:.1f} GB of fp32 traces per GPU vs 126 MB L2)"),
        "parallelism": f"dp{n_gpus} (trace-sharded; NCCL all-reduce of per-GPU totals)",
    }


# ------------------------------------------------------------------ product arm
def main_chase(args):
    import torch
    import torch.distributed as dist

    import paper_2303_02508_b200 as cb
    from paper_2303_02508_b200.parallel import reduce_sums, shard_bounds

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    w = inputs.workload(args.config, n_traces=args.traces)
    W = w.W
    if args.weak:   # weak scaling: every rank plans its own w.n_traces traces
        n_total = w.n_traces * world
    else:           # strong scaling (configs[4]): the workload's traces split across the ranks
        n_total = w.n_traces
    trace0, trace1 = shard_bounds(n_total, rank, world)
    n = trace1 - trace0
    x = torch.empty((n, w.ld), dtype=torch.float32, device=dev)
    inputs.synth_traces_device(x, w.n_steps, seed=w.seed, mode=w.mode, trace0=trace0)
    pid = None
    if len(w.profiles) > 1:
        pid = torch.empty(n, dtype=torch.uint8, device=dev)
        inputs.profile_ids_device(pid, seed=w.seed, n_profiles=len(w.profiles), trace0=trace0)
    per_prof = torch.tensor([w.interval_s * W * float(p.throughput_sps.min()) for p in w.profiles],
                            dtype=torch.float64, device=dev)
    J = per_prof[pid.long()] if pid is not None else per_prof[0].expand(n).contiguous()
    torch.cuda.synchronize()

    planner = cb.Planner(x, n_steps=w.n_steps, profiles=w.profiles, etas=w.etas, interval_s=w.interval_s,
                         history_len=w.history_len, profile_id=pid, job_samples=J, want_choice=True,
                         refit_stride=args.refit_stride, period_steps=args.period_steps, svr=svr_arg(args))

    def step():
        planner.run()
        if world > 1:
            reduce_sums(planner.sums)        # the one exchange step: NCCL all-reduce of chase_sum_t[n_eta]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    diag = planner.diag()
    sums0 = planner.sums.cpu().numpy()
    if diag.n_bad or sums0[0, 7] != n_total:
        raise RuntimeError(f"planner reported bad traces: n_bad={diag.n_bad}, n_ok={sums0[0, 7]}")

    stream = torch.cuda.current_stream(dev)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in kev:         # materialise the CUDA events before handing them to the library
        a.record(stream)
        b.record(stream)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # inputs smaller than a few L2s (C1-C3): the L2 is flushed between timed steps
    # (a 512 MB write outside each step's events), and the step time is the sum of
    # the per-step event times
    flush = (torch.empty(512 << 20, dtype=torch.uint8, device=dev)
             if l2_resident(w, n_total) else None)
    sev = ([(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
           if flush is not None else None)
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = cb.kernel_launches()
    clocks.begin()
    t0.record(stream)
    for k in range(args.steps):
        if flush is not None:
            flush.zero_()
            sev[k][0].record(stream)
        cb.set_kernel_events(*kev[k])
        step()
        if flush is not None:
            sev[k][1].record(stream)
    t1.record(stream)
    cb.set_kernel_events(None, None)
    torch.cuda.synchronize()
    clocks.end()
    if world > 1:
        dist.barrier()
    launches = cb.kernel_launches() - launches0
    clk = clocks.stop()

    elapsed_ms = t0.elapsed_time(t1) if flush is None else float(sum(a.elapsed_time(b) for a, b in sev))
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    tm = torch.tensor([elapsed_ms, kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    elapsed_ms, kern_ms = float(tm[0]), float(tm[1])
    ms_per_step = elapsed_ms / args.steps
    total_windows = float(n_total) * W
    value = total_windows / (ms_per_step / 1e3)

    R = args.refit_stride
    if svr_arg(args) is not None:
        peak, peak_src = fp64_peak()
        flops = svr_flops(w)
        achieved = flops / (kern_ms / 1e3) / 1e12
        roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": None, "kernel": planner_kernel_name(w, R, args.period_steps, {}),
                    "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms_per_step,
                    "algorithmic_flops_per_launch": flops, "flops_note": "lower bound: SMO iterations not counted",
                    "peak_source": peak_src}
    elif R == 0:
        peak, peak_src = measured_peaks()
        bpw = 4.0 + len(w.etas)   # fp32 trace value + one choice byte per eta (5 B for one eta)
        alg_bytes = n * W * bpw
        achieved = alg_bytes / (kern_ms / 1e3) / 1e9
        tpw = ncu_traffic_per_window(args.config if args.period_steps <= 1 else f"{args.config}_p{args.period_steps}")
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": None if tpw is None else tpw * n * W,
                    "kernel": planner_kernel_name(w, 0, args.period_steps),
                    "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms_per_step,
                    "algorithmic_bytes_per_launch": alg_bytes, "bytes_per_window": bpw,
                    "peak_source": peak_src}
    else:
        peak, peak_src = fp64_peak()
        fused = bool(diag.kernel_path & cb.PATH_ROLL_FUSED)
        flops = rolling_fused_flops(w, R) if fused else rolling_flops(w, R)
        achieved = flops / (kern_ms / 1e3) / 1e12
        tpw = ncu_traffic_per_window(f"{args.config}_roll{R}") if fused else None
        roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": None if tpw is None else tpw * n * W, "kernel": planner_kernel_name(w, R),
                    "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms_per_step,
                    "algorithmic_flops_per_launch": flops, "peak_source": peak_src,
                    "dram_bytes_per_window": tpw}

    latency = None
    if n_total <= 64 and world == 1:   # C1 / C2: one trace, latency-bound
        latency = bench_latency(planner, torch, stream, args.steps)

    # ---- e2e: the public host-buffer call, H2D of the inputs inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = bench_e2e(args, w, x, pid, J, cb, torch, dist, world, local, dev)

    cpu = None
    prefix_check = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, ns, dt = oracle_sample_rate(w, args.cpu_seconds, n, args.refit_stride, args.period_steps,
                                                 svr_arg(args))
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"first {ns} of {n} traces ({ns * W:.3g} windows, {dt:.1f} s on {cores} threads)"}
        if svr_arg(args) is None and not args.no_prefix_check:
            prefix_check = oracle_prefix_check(w, x, pid, J, ns, args, cb, torch)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded counter-based generator, inputs/)",
            "config": workload_config(w, world, args.refit_stride, args.period_steps, svr_arg(args),
                                      n_total=n_total, weak=args.weak),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "latency": latency,
            "gpu_launches": int(launches), "clocks": clk,
            "decisions_per_s": value * len(w.etas),
            "check": {"n_ok": float(sums0[0, 7]), "n_slow_windows": int(diag.n_slow_windows),
                      "kernel_path": int(diag.kernel_path), "oracle_prefix": prefix_check},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def l2_resident(w, n_total) -> bool:
    """Inputs + choices within 2 x the 126 MB L2 (C1, C2, C3): flush between steps."""
    return n_total * (w.ld * 4 + w.W * len(w.etas)) < 2 * 126e6


def bench_latency(planner, torch, stream, steps):
    """Latency-bound configs (one trace, C1/C2): the wall-clock microseconds of
    one chase_sweep call that returns its results (call + stream synchronize,
    host work included: argument checks, the cached tables, 8 kernel launches),
    the GPU time of the call by CUDA events, and the same call replayed as a
    CUDA graph (the launches captured once, stream-ordered)."""
    n = max(steps, 20)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        planner.run()
        torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / n * 1e6
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(n):
        planner.run()
    b.record(stream)
    torch.cuda.synchronize()
    gpu = a.elapsed_time(b) / n * 1e3
    out = {"us_per_call_wall": wall, "us_per_call_gpu_back_to_back": gpu, "calls": n}
    try:
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            planner.run()
        torch.cuda.current_stream().wait_stream(s2)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            planner.run()
        g.replay()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(n):
            g.replay()
            torch.cuda.synchronize()
        out["us_per_call_graph_wall"] = (time.perf_counter() - t) / n * 1e6
    except Exception as e:  # capture is an optimisation, not the contract
        out["graph_error"] = str(e)[:200]
    return out


def oracle_prefix_check(w, x, pid, J, ns, args, cb, torch, chunk=32768):
    """Parity of the whole cpu_baseline sample (untimed): the first `ns` traces of
    the benched workload planned by chase_sweep in the benched configuration
    (same kernels; choices and per-trace totals kept) against the oracle, chunk
    by chunk.  Choices must match bit for bit, and the per-trace totals too
    (the synthetic inputs are dyadic)."""
    import oracle
    W = w.W
    sub = x[:ns]
    pl = cb.Planner(sub, n_steps=w.n_steps, profiles=w.profiles, etas=w.etas, interval_s=w.interval_s,
                    history_len=w.history_len, profile_id=None if pid is None else pid[:ns],
                    job_samples=J[:ns].contiguous(), want_choice=True, want_per_trace=True,
                    refit_stride=args.refit_stride, period_steps=args.period_steps)
    res = pl.run()
    torch.cuda.synchronize()
    path = int(pl.diag().kernel_path)
    t0 = time.perf_counter()
    ch_bad = tot_bad = certified = 0
    first_bad = None
    # the fused rolling refit (sliding moments) is held to the tolerance contract: a choice may
    # differ only at a certified near-tie of the oracle's forecast
    tol = args.refit_stride > 0 and bool(path & cb.PATH_ROLL_FUSED)
    if tol:
        chunk = 2048
    for c0 in range(0, ns, chunk):
        m = min(chunk, ns - c0)
        tr = inputs.synth_traces_host(m, w.n_steps, seed=w.seed, mode=w.mode, trace0=c0)
        p_h = None if pid is None else pid[c0:c0 + m].cpu().numpy()
        o = oracle.plan_batch(tr, N=w.n_steps, L=w.history_len, T=w.T, refit_stride=args.refit_stride,
                              period=args.period_steps, profiles=w.profiles, profile_id=p_h, etas=w.etas,
                              delta=float(w.interval_s), job_samples=J[c0:c0 + m].cpu().numpy(),
                              want_forecast=tol, want_choice=True)
        g_ch = res.choice[:, c0:c0 + m, :W].cpu().numpy()
        if tol:
            for e, ii, ww in np.argwhere(g_ch != o["choice"]):
                p = w.profiles[0 if p_h is None else int(p_h[ii])]
                mc = float(np.max(tr[ii, :w.history_len]))
                c = sorted(oracle.cost(w.etas[e], p.avg_power_w[k], p.throughput_sps[k], float(p.limit_w[-1]), mc,
                                       o["forecast"][ii, ww]) for k in range(p.K))
                if c[1] - c[0] <= 1e-9 * abs(c[0]):
                    certified += 1
                    g_ch[e, ii, ww] = o["choice"][e, ii, ww]   # certified: counted, not a mismatch
        bad_rows = np.any(g_ch != o["choice"], axis=2)
        g_tot = res.per_trace[:, c0:c0 + m].cpu().numpy().view(cb.TOTALS_DTYPE).reshape(len(w.etas), m)
        if tol:   # totals of the traces whose choices agree, within 1e-9 (rounding order differs)
            ok_rows = ~np.any(res.choice[:, c0:c0 + m, :W].cpu().numpy() != o["choice"], axis=2)
            for f in ("time_s", "energy_j", "carbon_g", "samples"):
                a, b = g_tot[f][ok_rows], o["totals"][f][ok_rows]
                bad = np.abs(a - b) > 1e-9 * np.maximum(np.abs(b), 1e-300)
                tot_bad += int(bad.sum())
            tb = False
        else:
            tb = g_tot.tobytes() != o["totals"].tobytes()
        if tb:
            diff = np.any(g_tot.view(np.uint8).reshape(len(w.etas), m, 64) !=
                          o["totals"].view(np.uint8).reshape(len(w.etas), m, 64), axis=2)
            tot_bad += int(diff.sum())
            if first_bad is None:
                first_bad = c0 + int(np.argwhere(diff)[0][1])
        ch_bad += int(bad_rows.sum())
        if bad_rows.any() and first_bad is None:
            first_bad = c0 + int(np.argwhere(bad_rows)[0][1])
    del res, pl
    torch.cuda.empty_cache()
    return {"traces": int(ns), "windows": int(ns) * W * len(w.etas), "traces_with_choice_mismatch": ch_bad,
            "traces_with_totals_mismatch": tot_bad, "first_mismatch_trace": first_bad, "kernel_path": path,
            "certified_near_ties": certified if tol else None,
            "seconds": round(time.perf_counter() - t0, 1),
            "what": ("the cpu_baseline sample re-planned by chase_sweep (benched config) vs the oracle: "
                     + ("choices exact up to certified near-ties, per-trace totals within 1e-9 (tolerance "
                        "contract of the fused rolling refit)" if tol else
                        "choices bit-exact, per-trace totals bit-identical"))}


def bench_e2e(args, w, x, pid, J, cb, torch, dist, world, local, dev):
    """Same metric through chase_sweep_host: pinned HOST traces / ids / budgets,
    chunked H2D overlapping the fused kernels, host sums out."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 32 << 30
    row = w.ld * 4
    lws = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    n_e2e = args.e2e_traces or int(min(w.n_traces, avail * 0.3 / max(1, lws) / row))
    n_e2e = max(1024, (n_e2e // 1024) * 1024)
    n_e2e = min(n_e2e, w.n_traces)
    h = torch.empty((n_e2e, w.ld), dtype=torch.float32).pin_memory()
    h.copy_(x[:n_e2e])
    hp = None if pid is None else pid[:n_e2e].cpu().pin_memory()
    hJ = J[:n_e2e].cpu().pin_memory()
    chunk = min(n_e2e, 32768)
    ht = cb.make_traces(h, n_steps=w.n_steps, interval_s=w.interval_s)
    tc = cb.make_traces(h[:chunk], n_steps=w.n_steps, interval_s=w.interval_s)
    fcfg = cb.make_fcfg(interval_s=w.interval_s, history_len=w.history_len, refit_stride=args.refit_stride,
                        period_steps=args.period_steps, svr=svr_arg(args))
    ws = cb.alloc_workspace(cb.workspace_bytes(tc, fcfg, len(w.profiles), len(w.etas)), dev)
    stg = cb.alloc_workspace(cb.sweep_host_staging_bytes(ht, chunk, len(w.etas)), dev)

    def call():
        return cb.sweep_host(ht, fcfg, w.profiles, w.etas, chunk, stg, ws, h_profile_id=hp, h_job_samples=hJ)

    call()
    steps = max(2, min(args.steps, 5))
    stream = torch.cuda.current_stream(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(steps):
        sums = call()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    tm = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms = float(tm[0])
    if sums[0, 7] != n_e2e:
        raise RuntimeError(f"e2e sums report {sums[0, 7]} ok traces of {n_e2e}")
    h2d = n_e2e * (w.ld * 4 + (1 if hp is not None else 0) + 8)
    return {"value": n_e2e * w.W * world / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(len(w.etas) * 64), "traces_per_gpu": n_e2e, "ms_per_step": ms,
            "api": "chase_sweep_host (pinned host inputs, double-buffered H2D on a second stream)"}


MAPE_METRIC = "trace-windows evaluated/sec (walk-forward MAPE, linear + persistence)"


def main_mape(args):
    """Forecast-evaluation sweep (the Table 1 experiment,
    P:159-161, on synthetic traces): chase_forecast_mape over this GPU's traces.
    Roofline: HBM, 4 B per window (the trace value; 16 B per trace of output)."""
    import torch
    import torch.distributed as dist

    import paper_2303_02508_b200 as cb
    from paper_2303_02508_b200.parallel import shard_bounds

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    w = inputs.workload(args.config, n_traces=args.traces)
    n, W = w.n_traces, w.W
    trace0, _ = shard_bounds(n * world, rank, world)
    x = torch.empty((n, w.ld), dtype=torch.float32, device=dev)
    inputs.synth_traces_device(x, w.n_steps, seed=w.seed, mode=w.mode, trace0=trace0)
    t = cb.make_traces(x, n_steps=w.n_steps, interval_s=w.interval_s)
    sv = svr_arg(args)
    f = cb.make_fcfg(interval_s=w.interval_s, history_len=w.history_len, svr=sv)
    ws = cb.alloc_workspace(cb.workspace_bytes(t, f, 1, 1), dev)
    mp = torch.empty((n, 2), dtype=torch.float64, device=dev)
    st = torch.empty(n, dtype=torch.int32, device=dev)
    for _ in range(args.warmup):
        cb.forecast_mape(t, f, mp, ws, status=st)
    torch.cuda.synchronize()
    if int((st != 0).sum()) != 0:
        raise RuntimeError("forecast_mape reported invalid traces on the synthetic workload")
    stream = torch.cuda.current_stream(dev)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in kev:
        a.record(stream)
        b.record(stream)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = cb.kernel_launches()
    clocks.begin()
    t0.record(stream)
    for k in range(args.steps):
        cb.set_kernel_events(*kev[k])
        cb.forecast_mape(t, f, mp, ws, status=st)
    t1.record(stream)
    cb.set_kernel_events(None, None)
    torch.cuda.synchronize()
    clocks.end()
    if world > 1:
        dist.barrier()
    launches = cb.kernel_launches() - launches0
    clk = clocks.stop()
    tm = torch.tensor([t0.elapsed_time(t1), float(np.mean([a.elapsed_time(b) for a, b in kev]))],
                      dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms_per_step, kern_ms = float(tm[0]) / args.steps, float(tm[1])
    value = float(n) * W * world / (ms_per_step / 1e3)
    if sv is None:
        peak, peak_src = measured_peaks()
        alg = n * W * 4.0
        achieved = alg / (kern_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": None, "kernel": "mape_kernel (warp per trace, walk-forward predict + MAPE sums)",
                    "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms_per_step,
                    "algorithmic_bytes_per_launch": alg, "bytes_per_window": 4.0, "peak_source": peak_src}
    else:
        peak, peak_src = fp64_peak()
        flops = svr_flops(w)
        achieved = flops / (kern_ms / 1e3) / 1e12
        roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "traffic": None, "kernel": planner_kernel_name(w, 0, 0, sv) + " + mape_kernel",
                    "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms_per_step,
                    "algorithmic_flops_per_launch": flops, "flops_note": "lower bound: SMO iterations not counted",
                    "peak_source": peak_src}
    e2e = None
    if not args.no_e2e:   # host traces -> device (chunked, pinned) -> chase_forecast_mape -> host results
        chunk = min(n, 65536)
        h = torch.empty((chunk, w.ld), dtype=torch.float32).pin_memory()
        h.copy_(x[:chunk])
        hm = torch.empty((chunk, 2), dtype=torch.float64).pin_memory()
        xd = torch.empty_like(x[:chunk])
        tc = cb.make_traces(xd, n_steps=w.n_steps, interval_s=w.interval_s)
        wsc = cb.alloc_workspace(cb.workspace_bytes(tc, f, 1, 1), dev)
        mc = torch.empty((chunk, 2), dtype=torch.float64, device=dev)
        reps = max(1, n // chunk)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            xd.copy_(h, non_blocking=True)
            cb.forecast_mape(tc, f, mc, wsc)
            hm.copy_(mc, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        e2e = {"value": reps * chunk * W / (ms / 1e3), "unit": "trace-windows/s",
               "h2d_bytes_per_step": int(reps * chunk * w.ld * 4), "d2h_bytes_per_step": int(reps * chunk * 16),
               "api": "chase_forecast_mape on chunks copied from pinned host memory"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        ns = 256 if sv is None else 16
        tr_h = inputs.synth_traces_host(ns, w.n_steps, seed=w.seed, mode=w.mode)
        t_0 = time.perf_counter()
        _, _, cores = oracle.evaluate_batch(tr_h, N=w.n_steps, L=w.history_len, T=w.T, svr=sv)
        dt = time.perf_counter() - t_0
        ns = int(min(n, ns * max(1.0, args.cpu_seconds / max(dt, 1e-3))))
        tr_h = inputs.synth_traces_host(ns, w.n_steps, seed=w.seed, mode=w.mode)
        t_0 = time.perf_counter()
        _, _, cores = oracle.evaluate_batch(tr_h, N=w.n_steps, L=w.history_len, T=w.T, svr=sv)
        dt = time.perf_counter() - t_0
        cpu = {"value": ns * W / dt, "unit": "trace-windows/s", "cores": cores, "kind": "oracle",
               "sample": f"first {ns} of {n} traces ({ns * W:.3g} windows, {dt:.1f} s on {cores} threads)"}
    if rank == 0:
        cfg = workload_config(w, world, 0, 0, sv)
        cfg["workload"] = f"{w.name} traces, walk-forward forecast evaluation (Table 1 shape, P:159-161)"
        line = {"metric": MAPE_METRIC, "value": value, "unit": "trace-windows/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded counter-based generator, inputs/)", "config": cfg,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk, "check": {"mean_mape_linear": float(mp[:, 0].mean()),
                                         "mean_mape_persistence": float(mp[:, 1].mean())}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


TIMELINE_METRIC = "trace-windows audited/sec (per-period timeline rows of the planned replay)"


def main_timeline(args):
    """Timeline / audit rows: chase_timeline over this GPU's
    traces after one planning sweep (choices + decision forecasts kept).
    Roofline: HBM, per window 4 B trace + 1 B choice + 8 B forecast read, plus
    64 B per row written."""
    import torch

    import paper_2303_02508_b200 as cb

    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    w = inputs.workload(args.config, n_traces=args.traces or 100_000)
    n, W = w.n_traces, w.W
    P = max(args.period_steps, 1)
    x = torch.empty((n, w.ld), dtype=torch.float32, device=dev)
    inputs.synth_traces_device(x, w.n_steps, seed=w.seed, mode=w.mode, trace0=rank * n)
    J = torch.full((n,), float(w.interval_s * W * w.profiles[0].throughput_sps.min()), dtype=torch.float64,
                   device=dev)
    pl = cb.Planner(x, n_steps=w.n_steps, profiles=w.profiles[:1], etas=w.etas[:1], job_samples=J, want_choice=True,
                    want_forecast=True, period_steps=P)
    res = pl.run()
    n_per = -(-W // P)
    rows = torch.empty((n, n_per, 8), dtype=torch.float64, device=dev)
    t = cb.make_traces(x, n_steps=w.n_steps, interval_s=w.interval_s)
    ws = cb.alloc_workspace(cb.workspace_bytes(t, cb.make_fcfg(), 1, 1), dev)

    def step():
        cb.timeline(t, w.history_len, w.profiles[:1], rows, n, ws, period_steps=P, choice=res.choice[0],
                    ld_c=pl.ld_c, forecast=res.forecast, ld_f=pl.ld_f, job_samples=J)

    for _ in range(args.warmup):
        step()
    stream = torch.cuda.current_stream(dev)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in kev:
        a.record(stream)
        b.record(stream)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize()
    launches0 = cb.kernel_launches()
    clocks.begin()
    t0.record(stream)
    for k in range(args.steps):
        cb.set_kernel_events(*kev[k])
        step()
    t1.record(stream)
    cb.set_kernel_events(None, None)
    torch.cuda.synchronize()
    clocks.end()
    launches = cb.kernel_launches() - launches0
    clk = clocks.stop()
    ms_per_step = t0.elapsed_time(t1) / args.steps
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    alg = n * W * 13.0 + n * n_per * 64.0
    peak, peak_src = measured_peaks()
    achieved = alg / (kern_ms / 1e3) / 1e9
    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        fc, ch = res.forecast.cpu().numpy(), res.choice.cpu().numpy()[0]
        xs = x[:2000].cpu().numpy().astype(np.float64)
        p0 = w.profiles[0]
        t_0 = time.perf_counter()
        ns = 0
        while time.perf_counter() - t_0 < min(args.cpu_seconds, 5.0) and ns < 2000:
            oracle.timeline(xs[ns, :w.n_steps], L=w.history_len, period=P, choice=ch[ns, :W], forecast=fc[ns, :W],
                            limit_w=p0.limit_w, avg_power=p0.avg_power_w, thr=p0.throughput_sps,
                            delta=float(w.interval_s), J=float(J[ns]))
            ns += 1
        dt = time.perf_counter() - t_0
        cpu = {"value": ns * W / dt, "unit": "trace-windows/s", "cores": 1, "kind": "oracle",
               "sample": f"first {ns} traces, one thread ({dt:.1f} s)"}
    cfg = workload_config(w, 1, 0, P)
    cfg["workload"] = f"{w.name} traces: per-period audit rows of the planned replay (SPEC emit_timeline)"
    line = {"metric": TIMELINE_METRIC, "value": float(n) * W / (ms_per_step / 1e3), "unit": "trace-windows/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded counter-based generator, inputs/)", "config": cfg,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "kernel": "timeline_kernel (warp per trace, lane per period)",
                         "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms_per_step,
                         "algorithmic_bytes_per_launch": alg, "peak_source": peak_src},
            "cpu_baseline": cpu, "e2e": None, "gpu_launches": int(launches), "clocks": clk,
            "check": {"rows": int(n * n_per)}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    args = parse_args(argv)
    if args.impl == "reference":
        return main_reference(args)
    if args.mode == "mape":
        return main_mape(args)
    if args.mode == "timeline":
        return main_timeline(args)
    return main_chase(args)


if __name__ == "__main__":
    sys.exit(main())
