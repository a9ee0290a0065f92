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


def combine_totals(t64_list):
    """Reduce a list of int64 [n_policies, 24] totals tensors (e.g. of consecutive chunks) into a new tensor:
    sums (wrapping), the makespan maximum, the OR of the error flags."""
    import torch

    allt = torch.stack(list(t64_list))
    red = allt.sum(dim=0)
    red[:, MAX_FIELD] = allt[:, :, MAX_FIELD].max(dim=0).values
    flags = allt[0, :, OR_FIELD].clone()
    for r in range(1, allt.shape[0]):
        flags |= allt[r, :, OR_FIELD]
    red[:, OR_FIELD] = flags
    return red


def simulate_generated(g, cfg, pols, trace_id0, n, chunk=1 << 22, sample_stride=0, device=None, stream=None,
                       on_chunk=None):
    """Generate the config's traces [trace_id0, trace_id0 + n) on the device chunk by chunk (SURVEY.md §8(d) C5:
    chunks of 2^22 traces, so 10^8 traces run on any number of GPUs) and simulate each chunk with one mig_simulate
    call. Returns (totals int64 [n_policies, 24] on the device, summed over the chunks; sampled results uint8
    [n_samples * n_policies, 96] of the trace ids that are multiples of sample_stride, or None).

    Only the chunk loop lives here: generation is tracegen's (the seeded input generator), every step of the
    method runs in libmig's kernels."""
    import torch

    import paper_2508_18556_b200 as mig
    from tracegen import tracegen as tg

    dev = device or torch.device("cuda", torch.cuda.current_device())
    seed = tg.seed_of(cfg)
    J = tg.jobs_per_trace(cfg)
    n_pol = len(pols)
    tots, samples = [], []
    tot = torch.empty((n_pol, 192), dtype=torch.uint8, device=dev)
    for c0 in range(0, n, chunk):
        m = min(chunk, n - c0)
        t0 = trace_id0 + c0
        jobs, ext, off = tg.generate_device(cfg, m, trace_id0=t0, seed=seed, device=dev, stream=stream)
        tr = mig.Traces(jobs, ext, off, m, seed=seed, trace_id0=t0, max_jobs=J,
                        flags=0 if tg.CONFIG_HAS_DYNAMIC[cfg] else mig.MIG_TRACES_NO_DYNAMIC)
        res, _ = mig.mig_simulate(g, tr, pols, out=None, totals=tot, write_results=sample_stride > 0, stream=stream)
        tots.append(tot.view(torch.int64).view(n_pol, N_FIELDS).clone())
        if sample_stride:
            first = (-t0) % sample_stride  # first id >= t0 that is a multiple of the stride
            if first < m:
                rows = torch.arange(first, m, sample_stride, device=dev)
                samples.append(res.view(m, n_pol, 96)[rows].reshape(-1, 96))
        if on_chunk is not None:
            on_chunk(c0, m)
        del jobs, ext, off, tr, res
    red = combine_totals(tots)
    return red, (torch.cat(samples) if samples else None)
