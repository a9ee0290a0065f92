"""Trace sharding and the cross-GPU metric reduce.

Traces are independent: rank r of W simulates global trace ids [r*N, (r+1)*N) (weak scaling) or
[r*N/W, (r+1)*N/W) (strong scaling) with no data-path exchange. The only exchange step is the per-policy metric
reduce of north_star: the int64 totals (mig_policy_totals, 20 fields per policy) are summed over ranks, except the
makespan maximum and the error flags, which are max-reduced. Integer sums are exact in any order, so the reduced
totals are bit-identical for any W.
"""
from __future__ import annotations

N_FIELDS = 24
MAX_FIELDS = (13, 20)  # makespan_max, error_flags


def shard_range(rank: int, world: int, n_per_rank: int = 0, n_total: int = 0):
    """(trace_id0, n) of this rank: weak scaling with n_per_rank, else strong scaling over n_total."""
    if n_per_rank:
        return rank * n_per_rank, n_per_rank
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi - lo


def reduce_totals(t64, dist, group=None):
    """In-place all_reduce of an int64 [n_policies, 24] totals tensor (NCCL over NVLink, or gloo on CPU)."""
    mx = t64[:, list(MAX_FIELDS)].clone()
    dist.all_reduce(t64, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    for k, f in enumerate(MAX_FIELDS):
        t64[:, f] = mx[:, k]
    return t64
