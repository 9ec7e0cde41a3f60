"""Run one planner call per workload, twice each (the second is the one to
capture), for a single `ncu` command over several configs or period lengths:

  ncu --set full -k regex:sweep --launch-skip-before-match 0 ... python tools/ncu_workloads.py configs
  ncu ... python tools/ncu_workloads.py periods

configs: C1, C2, C3, C4 (bench.py's inputs); periods: C5 at P = 2, 3, 24, 168.
Tuning/profiling only (not a test, not the bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2303_02508_b200 as cb  # noqa: E402


def planner(name, period=0):
    w = inputs.workload(name)
    x = torch.empty((w.n_traces, w.ld), dtype=torch.float32, device="cuda")
    inputs.synth_traces_device(x, w.n_steps, seed=w.seed, mode=w.mode)
    pid = None
    if len(w.profiles) > 1:
        pid = torch.empty(w.n_traces, dtype=torch.uint8, device="cuda")
        inputs.profile_ids_device(pid, seed=w.seed, n_profiles=len(w.profiles))
    per_prof = torch.tensor([w.interval_s * w.W * float(p.throughput_sps.min()) for p in w.profiles],
                            dtype=torch.float64, device="cuda")
    J = per_prof[pid.long()] if pid is not None else per_prof[0].expand(w.n_traces).contiguous()
    return cb.Planner(x, n_steps=w.n_steps, profiles=w.profiles, etas=w.etas, interval_s=w.interval_s,
                      history_len=w.history_len, profile_id=pid, job_samples=J, want_choice=True,
                      period_steps=period), x


jobs = [("C1", 0), ("C2", 0), ("C3", 0), ("C4", 0)] if sys.argv[1] == "configs" else \
       [("C5", 2), ("C5", 3), ("C5", 24), ("C5", 168)]
for name, period in jobs:
    pl, x = planner(name, period)
    for _ in range(2):
        pl.run()
    torch.cuda.synchronize()
    print(name, period, "path", pl.diag().kernel_path, flush=True)
    del pl, x
    torch.cuda.empty_cache()
