"""The N > 1 path through libchase (BASELINE configs[4]):
two ranks, each on cuda:0 (this box has one GPU), gloo on CUDA tensors for the
one exchange step.  Each rank generates its contiguous shard of a C5-shaped
workload with its own trace offset (as bench.py's ranks do), runs the real
chase_sweep on it, and reduces the per-rank totals with parallel.reduce_sums
(all_reduce and the deterministic rank-order gather).  The reduced totals must
equal the unsharded GPU sweep's and the oracle's.

The ranks never wait on each other inside a kernel: the only coupling is the
host-side gloo collective after each rank's stream has finished.

The log prints, per rank, the chase_sweep call (CUDA events around the whole
call), the sweep kernel alone (chase_set_kernel_events) and the all-reduce: at
1.25e5 traces per GPU (configs[4] on 8 GPUs) the per-call overheads (upload,
fit, finalize, sums) become visible next to the sweep."""
import json
import os
import socket
import tempfile

import numpy as np
import pytest

import inputs
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

N_TOTAL = 250_000          # 2 ranks x 1.25e5 traces (configs[4]'s per-GPU share at G = 8)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _workload():
    return inputs.workload("C5", n_traces=N_TOTAL)


def _rank_main(rank, world, port, outdir):
    import paper_2303_02508_b200 as cb
    from paper_2303_02508_b200.parallel import reduce_sums, shard_bounds
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = _workload()
        t0, t1 = shard_bounds(w.n_traces, rank, world)
        n = t1 - t0
        dev = torch.device("cuda", 0)
        x = torch.empty((n, w.ld), dtype=torch.float32, device=dev)
        inputs.synth_traces_device(x, w.n_steps, seed=w.seed, mode=w.mode, trace0=t0)
        J = torch.full((n,), float(w.job_samples()[0]), dtype=torch.float64, device=dev)
        pl = cb.Planner(x, n_steps=w.n_steps, profiles=w.profiles, etas=w.etas, job_samples=J, want_choice=True)
        pl.run()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        for e in ev:
            e.record()
        torch.cuda.synchronize()
        cb.set_kernel_events(ev[2], ev[3])
        ev[0].record()
        pl.run()
        ev[1].record()
        cb.set_kernel_events(None, None)
        torch.cuda.synchronize()          # the rank's stream is done before the host collective
        local = pl.sums.clone()
        dist.barrier()
        ev[4].record()
        a = reduce_sums(pl.sums)          # all_reduce(SUM) on the CUDA tensor (gloo)
        ev[5].record()
        torch.cuda.synchronize()
        b = reduce_sums(local.clone(), deterministic=True)
        d = pl.diag()
        np.save(os.path.join(outdir, f"r{rank}.npy"),
                np.stack([a.cpu().numpy(), b.cpu().numpy(), local.cpu().numpy()]))
        with open(os.path.join(outdir, f"t{rank}.json"), "w") as f:
            json.dump({"rank": rank, "traces": [t0, t1], "call_ms": ev[0].elapsed_time(ev[1]),
                       "sweep_kernel_ms": ev[2].elapsed_time(ev[3]), "allreduce_ms": ev[4].elapsed_time(ev[5]),
                       "kernel_path": int(d.kernel_path), "n_bad": int(d.n_bad)}, f)
    finally:
        dist.destroy_process_group()


def test_two_ranks_through_libchase_equal_unsharded_gpu_and_oracle():
    import paper_2303_02508_b200 as cb
    world = 2
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_rank_main, args=(world, port, d), nprocs=world, join=True, start_method="spawn")
        res = [np.load(os.path.join(d, f"r{r}.npy")) for r in range(world)]
        tim = [json.load(open(os.path.join(d, f"t{r}.json"))) for r in range(world)]
    for t in tim:
        print("rank timing:", json.dumps(t))
        print(f"  per-call overhead outside the sweep kernel: {t['call_ms'] - t['sweep_kernel_ms']:.3f} ms "
              f"({100 * (1 - t['sweep_kernel_ms'] / t['call_ms']):.1f}% of the call)")
        assert t["kernel_path"] & cb.PATH_HEADLINE and t["n_bad"] == 0
    w = _workload()
    # unsharded GPU sweep of the same traces
    dev = torch.device("cuda", 0)
    x = torch.empty((w.n_traces, w.ld), dtype=torch.float32, device=dev)
    inputs.synth_traces_device(x, w.n_steps, seed=w.seed, mode=w.mode)
    J = torch.full((w.n_traces,), float(w.job_samples()[0]), dtype=torch.float64, device=dev)
    pl = cb.Planner(x, n_steps=w.n_steps, profiles=w.profiles, etas=w.etas, job_samples=J, want_choice=False)
    full_gpu = pl.run().sums.cpu().numpy()
    del x
    # the oracle on the host, unsharded
    tr = inputs.synth_traces_host(w.n_traces, w.n_steps, seed=w.seed, mode=w.mode)
    full_o = oracle.plan_batch(tr, N=w.n_steps, L=w.history_len, T=w.T, profiles=w.profiles, etas=w.etas,
                               job_samples=w.job_samples(), want_forecast=False, want_choice=False)["sums"]
    assert full_o[0, 7] == w.n_traces
    for r in range(world):
        allred, determ, local = res[r]
        assert np.array_equal(determ, res[0][1])                       # bitwise identical on every rank
        np.testing.assert_allclose(allred, full_gpu, rtol=1e-12, atol=0)
        np.testing.assert_allclose(determ, full_gpu, rtol=1e-12, atol=0)
        np.testing.assert_allclose(allred, full_o, rtol=1e-9, atol=0)
        assert allred[0, 7] == w.n_traces
    assert res[0][2][0, 7] + res[1][2][0, 7] == w.n_traces and 0 < res[0][2][0, 7] < w.n_traces
