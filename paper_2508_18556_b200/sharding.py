"""Trace sharding and the cross-GPU metric reduce.

Traces are independent: rank r of W simulates global trace ids [r*N, (r+1)*N) (weak scaling) or
[r*N/W, (r+1)*N/W) (strong scaling) with no data-path exchange. The only exchange step is the per-policy metric
reduce of north_star: one all_gather of every rank's int64 totals (mig_policy_totals, 24 fields per policy, 192 B
per policy: latency-bound over NVLink / NVSwitch), then a local reduce on the device: fields are summed (wrapping,
like the decision-hash sum), the makespan maximum is max-reduced and the error flags OR-ed (NCCL has no bitwise-OR
reduction, and a MAX would drop flags set on different ranks). Integer sums are exact in any order, so the reduced
totals are bit-identical for any W.
"""
from __future__ import annotations

N_FIELDS = 24
MAX_FIELD = 13  # makespan_max
OR_FIELD = 20  # error_flags


def shard_range(rank: int, world: int, n_per_rank: int = 0, n_total: int = 0):
    """(trace_id0, n) of this rank: weak scaling with n_per_rank, else strong scaling over n_total."""
    if n_per_rank:
        return rank * n_per_rank, n_per_rank
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi - lo


def reduce_totals(t64, dist, group=None):
    """In-place reduce over ranks of an int64 [n_policies, 24] totals tensor (NCCL over NVLink, or gloo on CPU):
    one all_gather, then sum / max / bitwise-or per field on the tensor's device."""
    import torch

    world = dist.get_world_size(group)
    parts = [torch.empty_like(t64) for _ in range(world)]
    dist.all_gather(parts, t64.contiguous(), group=group)
    allt = torch.stack(parts)  # [world, n_policies, 24]
    red = allt.sum(dim=0)
    red[:, MAX_FIELD] = allt[:, :, MAX_FIELD].max(dim=0).values
    flags = allt[0, :, OR_FIELD].clone()
    for r in range(1, world):
        flags |= allt[r, :, OR_FIELD]
    red[:, OR_FIELD] = flags
    t64.copy_(red)
    return t64
