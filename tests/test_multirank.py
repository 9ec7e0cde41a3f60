"""Multi-GPU host logic on CPU: contiguous trace
sharding + the one all-reduce of per-rank totals, world_size 2 over gloo.

Each rank plans ONLY its shard (generated with its own trace offset, as the
bench's ranks do on their GPUs), with the oracle standing in for the per-rank
chase_sweep (this is a CPU test of the host logic); the reduced totals must
equal the unsharded oracle's.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle
from paper_2303_02508_b200.parallel import percentages, reduce_sums, shard_bounds

N_TRACES, N_STEPS, SEED = 203, 24 + 600, 11


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _workload():
    w = inputs.workload("C4", n_traces=N_TRACES)
    w.n_steps, w.seed, w.etas = N_STEPS, SEED, [0.3, 0.5]
    return w


def _plan(w, t0, t1):
    n = t1 - t0
    tr = inputs.synth_traces_host(n, w.n_steps, seed=w.seed, mode=w.mode, trace0=t0)
    pid = inputs.profile_ids_host(n, seed=w.seed, n_profiles=len(w.profiles), trace0=t0)
    J = w.job_samples(pid)
    return oracle.plan_batch(tr, N=w.n_steps, L=w.history_len, T=w.T, profiles=w.profiles, profile_id=pid,
                             etas=w.etas, delta=float(w.interval_s), job_samples=J, want_forecast=False,
                             want_choice=False, threads=1)


def _rank_main(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = _workload()
        t0, t1 = shard_bounds(w.n_traces, rank, world)
        local = torch.from_numpy(_plan(w, t0, t1)["sums"].copy())
        a = reduce_sums(local.clone())
        b = reduce_sums(local.clone(), deterministic=True)
        np.save(os.path.join(outdir, f"r{rank}.npy"), np.stack([a.numpy(), b.numpy(), local.numpy()]))
        np.save(os.path.join(outdir, f"b{rank}.npy"), np.array([t0, t1]))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_partition():
    for n in (0, 1, 7, 203, 10**6):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_percentages_match_spec_formula():
    # corrected two-period golden: 33.226811% / 13.559322% / 13.333333%
    row = [5400.0, 1215000.0, 971 / 8, 0, 81000 / 17, 295 * 3600 * 45 / 34, 24721 / 136, 1]
    p = percentages(row)
    assert abs(p["carbon_reduction_pct"] - 33.226811) < 1e-5
    assert abs(p["time_increase_pct"] - 13.333333) < 1e-5
    assert abs(p["energy_reduction_pct"] - 13.559322) < 1e-5


def test_two_rank_gloo_sharded_totals_equal_unsharded_oracle():
    world = 2
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_rank_main, args=(world, port, d), nprocs=world, join=True, start_method="spawn")
        res = [np.load(os.path.join(d, f"r{r}.npy")) for r in range(world)]
        bounds = [tuple(np.load(os.path.join(d, f"b{r}.npy"))) for r in range(world)]
    w = _workload()
    full = _plan(w, 0, w.n_traces)["sums"]
    assert bounds == [shard_bounds(w.n_traces, r, world) for r in range(world)]
    assert full[:, 7].tolist() == [float(w.n_traces)] * len(w.etas)       # every trace valid
    for r in range(world):
        allred, determ, local = res[r]
        # the shards' local totals add up to the unsharded totals ...
        assert np.array_equal(determ, res[0][1])                           # bitwise on every rank
        assert np.allclose(allred, full, rtol=1e-12, atol=0)
        assert np.allclose(determ, full, rtol=1e-12, atol=0)
        assert allred[:, 7].tolist() == full[:, 7].tolist()                # counts exact
    # ... and the shards really were disjoint halves
    assert np.allclose(res[0][2] + res[1][2], full, rtol=1e-12, atol=0)
    assert res[0][2][0, 7] + res[1][2][0, 7] == w.n_traces
    assert 0 < res[0][2][0, 7] < w.n_traces
