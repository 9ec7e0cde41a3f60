"""Trace sharding across GPUs and the one exchange step.

Traces are independent (the planner couples windows only within a trace), so
rank r of G plans its own contiguous range of traces with no data-path
collective; the only exchange is the sum of the per-GPU totals
`chase_sum_t[n_eta]` (8 f64 per eta: time, energy, carbon, samples, the three
baseline totals and the count of status-0 traces).

Host-side logic only: the per-rank sweep itself is `chase_sweep`.
"""
from __future__ import annotations


def shard_bounds(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Rank r's traces [floor(r*n/G), floor((r+1)*n/G)): contiguous, balanced
    to within one trace, covering [0, n) exactly once."""
    if world < 1 or not 0 <= rank < world or n_total < 0:
        raise ValueError(f"bad shard request: n={n_total} rank={rank} world={world}")
    return (rank * n_total) // world, ((rank + 1) * n_total) // world


def reduce_sums(sums, *, group=None, deterministic: bool = False):
    """Sum the per-rank totals `sums` ([n_eta][8] f64 tensor, in place) over the
    process group.  NCCL for CUDA tensors (the bench), gloo for CPU tensors
    (tests).  deterministic=True gathers every rank's totals and adds them in
    rank order, so the result is bitwise identical on every rank and for every
    run (SURVEY §8(e) option 1); the default is one all_reduce(SUM)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return sums
    world = dist.get_world_size(group)
    if world == 1:
        return sums
    if not deterministic:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
        return sums
    if sums.is_cuda and dist.get_backend(group) != "nccl":
        # gloo gathers host tensors only: gather a host copy, write the result back
        host = sums.cpu()
        reduce_sums(host, group=group, deterministic=True)
        sums.copy_(host)
        return sums
    parts = [torch.empty_like(sums) for _ in range(world)]
    dist.all_gather(parts, sums.contiguous(), group=group)
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    sums.copy_(acc)
    return sums


def percentages(sums_row):
    """S:382 comparison of one eta's global totals: carbon and energy reduction
    = 100*(base - aware)/base, time increase = 100*(aware - base)/base."""
    t, e, c = float(sums_row[0]), float(sums_row[1]), float(sums_row[2])
    bt, be, bc = float(sums_row[4]), float(sums_row[5]), float(sums_row[6])
    return {
        "carbon_reduction_pct": 100.0 * (bc - c) / bc if bc else 0.0,
        "energy_reduction_pct": 100.0 * (be - e) / be if be else 0.0,
        "time_increase_pct": 100.0 * (t - bt) / bt if bt else 0.0,
    }
