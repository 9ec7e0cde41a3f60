"""Closed-form period horizons: how many full periods the closed form decides
(chase_diag_t.n_seq_periods counts the ones it declined), on C5-shaped traces."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import inputs
import paper_2303_02508_b200 as cb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
w = inputs.workload("C5", n_traces=n)
tr = inputs.synth_traces_host(n, w.n_steps, seed=5)
x = torch.from_numpy(tr).cuda()
for P in (2, 3, 5, 12, 24, 168, 720):
    pl = cb.Planner(x, n_steps=w.n_steps, profiles=w.profiles, etas=w.etas, history_len=24, period_steps=P,
                    want_choice=False, want_forecast=False)
    pl.run()
    torch.cuda.synchronize()
    d = pl.diag()
    full = n * ((w.n_steps - 24) // P)
    print(f"P={P} full_periods={full} n_seq={d.n_seq_periods} ({d.n_seq_periods / full:.4f}) n_slow={d.n_slow_windows} "
          f"path={d.kernel_path}")
