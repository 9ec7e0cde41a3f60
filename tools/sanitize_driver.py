#!/usr/bin/env python3
"""A small workload for compute-sanitizer (memcheck / racecheck / synccheck,
one tool per run): the headline kernel, the decision-period instantiations,
the general multi-eta kernel, the fused rolling refit, the forecast-first
paths, the timeline and MAPE kernels, the host-input sweep -- on C1 and a
257-trace C4 slice, each checked against the oracle so a silent corruption
fails the run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_2303_02508_b200 as cb  # noqa: E402

DEV = torch.device("cuda:0")


def plan(w, tr, pid, etas, **kw):
    x = torch.from_numpy(tr).to(DEV)
    J = w.job_samples(pid)
    pl = cb.Planner(x, n_steps=w.n_steps, profiles=w.profiles, etas=etas,
                    profile_id=None if pid is None else torch.from_numpy(pid).to(DEV),
                    job_samples=torch.from_numpy(J).to(DEV), want_choice=True, want_per_trace=True, **kw)
    res = pl.run()
    torch.cuda.synchronize()
    return res, pl.diag(), J


def main():
    cases = []
    c1 = inputs.workload("C1")
    c4 = inputs.workload("C4", n_traces=257)
    c4.n_steps = 24 + 2500
    for w in (c1, c4):
        tr = inputs.synth_traces_host(w.n_traces, w.n_steps, seed=w.seed, mode=w.mode)
        pid = (inputs.profile_ids_host(w.n_traces, seed=w.seed, n_profiles=len(w.profiles))
               if len(w.profiles) > 1 else None)
        for name, etas, kw, okw in (
                ("headline", [0.5], {}, {}),
                ("general-multi-eta", [0.0, 0.5, 1.0], {}, {}),
                ("forecast-out", [0.5], dict(want_forecast=True), {}),
                ("periods-2", [0.5], dict(period_steps=2), dict(period=2)),
                ("periods-24", [0.5], dict(period_steps=24), dict(period=24)),
                ("periods-168", [0.5], dict(period_steps=168), dict(period=168)),
                ("rolling-fused-1", [0.5], dict(refit_stride=1), dict(refit_stride=1)),
                ("rolling-fused-24", [0.5], dict(refit_stride=24), dict(refit_stride=24)),
                ("rolling-exact", [0.5], dict(refit_stride=1, want_forecast=True), dict(refit_stride=1)),
        ):
            res, d, J = plan(w, tr, pid, etas, **kw)
            o = oracle.plan_batch(tr, N=w.n_steps, L=w.history_len, T=w.T, profiles=w.profiles, profile_id=pid,
                                  etas=etas, job_samples=J, **okw)
            g = res.choice.cpu().numpy()[:, :, :w.W]
            mism = int((g != o["choice"]).sum())
            tol = "rolling-fused" in name
            assert (mism <= 2) if tol else mism == 0, (w.name, name, mism)
            np.testing.assert_allclose(res.sums.cpu().numpy(), o["sums"], rtol=1e-9 if not tol else 1e-6)
            cases.append(f"{w.name}:{name}:path={d.kernel_path}:slow={d.n_slow_windows}")
        # timeline + MAPE + host sweep
        x = torch.from_numpy(tr).to(DEV)
        t = cb.make_traces(x, n_steps=w.n_steps)
        f = cb.make_fcfg()
        ws = cb.alloc_workspace(cb.workspace_bytes(t, f, len(w.profiles), 1), DEV)
        mp = torch.empty((w.n_traces, 2), dtype=torch.float64, device=DEV)
        cb.forecast_mape(t, f, mp, ws)
        res, d, J = plan(w, tr, pid, [0.5], want_forecast=True)
        rows = torch.empty((w.n_traces, w.W, 8), dtype=torch.float64, device=DEV)
        cb.timeline(t, w.history_len, w.profiles, rows, w.n_traces, ws, choice=res.choice[0], ld_c=res.choice.shape[2],
                    forecast=res.forecast, ld_f=res.forecast.shape[1],
                    profile_id=None if pid is None else torch.from_numpy(pid).to(DEV),
                    job_samples=torch.from_numpy(J).to(DEV))
        h = torch.from_numpy(tr).pin_memory()
        ht = cb.make_traces(h, n_steps=w.n_steps)
        chunk = max(1, w.n_traces // 3)
        tc = cb.make_traces(h[:chunk], n_steps=w.n_steps)
        ws2 = cb.alloc_workspace(cb.workspace_bytes(tc, f, len(w.profiles), 1), DEV)
        stg = cb.alloc_workspace(cb.sweep_host_staging_bytes(ht, chunk, 1), DEV)
        sums = cb.sweep_host(ht, f, w.profiles, [0.5], chunk, stg, ws2,
                             h_profile_id=None if pid is None else torch.from_numpy(pid).pin_memory(),
                             h_job_samples=torch.from_numpy(J).pin_memory())
        torch.cuda.synchronize()
        assert sums[0, 7] == w.n_traces
        cases.append(f"{w.name}:timeline+mape+host-sweep")
    print("sanitize driver OK:", len(cases), "cases;", "; ".join(cases))


if __name__ == "__main__":
    main()
