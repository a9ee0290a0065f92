"""Multi-GPU path on CPU: world_size 2 over gloo. Each rank takes its shard of traces (sharding.shard_range),
computes its per-policy totals (with the oracle, since there is no GPU here), and runs the same reduce_totals the
bench runs over NCCL. The reduced totals must equal the single-process totals bit for bit."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import geom_path

CFG, N_TOTAL = 3, 64


def totals_of(res):
    """mig_policy_totals layout (24 u64) from per-trace results [n_traces, n_pol]."""
    n_pol = res.shape[1]
    t = np.zeros((n_pol, 24), np.uint64)
    for p in range(n_pol):
        r = res[:, p]
        t[p, 0] = len(r)
        for k, f in enumerate(["n_jobs", "completed", "rejected", "failed", "ooms", "preempts", "restarts",
                               "placements", "waits", "creates", "destroys"]):
            t[p, 1 + k] = r[f].astype(np.uint64).sum()
        t[p, 12] = r["makespan"].astype(np.uint64).sum()
        t[p, 13] = r["makespan"].max(initial=0)
        t[p, 14] = r["energy_wticks"].sum(dtype=np.uint64)
        t[p, 15] = r["turnaround_sum"].sum(dtype=np.uint64)
        t[p, 16] = r["busy_slice_ticks"].sum(dtype=np.uint64)
        t[p, 17] = r["decision_hash"].sum(dtype=np.uint64)
        t[p, 18] = r["mem_mib_ticks"].sum(dtype=np.uint64)
        t[p, 19] = r["wasted_ticks"].sum(dtype=np.uint64)
    return t


def shard_totals(t0, n):
    from oracle import oracle as orc
    from tracegen import tracegen as tg

    jobs, ext, off = tg.generate_host(CFG, n, trace_id0=t0)
    g = orc.Geometry(geom_path(tg.CONFIG_GEOMETRY[CFG]))
    pols = [orc.policy(kind=3, flags=1), orc.policy(kind=3), orc.policy(kind=0)]
    res = orc.simulate(g, jobs, ext, off, pols, seed=tg.seed_of(CFG), trace_id0=t0)
    return totals_of(res)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_18556_b200.sharding import reduce_totals, shard_range

    t0, n = shard_range(rank, world, n_total=N_TOTAL)
    t = torch.from_numpy(shard_totals(t0, n).view(np.int64).copy())
    reduce_totals(t, dist)
    if rank == 0:
        out.put(t.numpy().view(np.uint64).copy())
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_and_reduce_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = shard_totals(0, N_TOTAL)
    assert np.array_equal(got, want)


def test_shard_ranges():
    from paper_2508_18556_b200.sharding import shard_range

    assert [shard_range(r, 4, n_total=10) for r in range(4)] == [(0, 2), (2, 3), (5, 2), (7, 3)]
    assert shard_range(3, 8, n_per_rank=1000) == (3000, 1000)


def _flags_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_18556_b200.sharding import reduce_totals

    t = torch.zeros((2, 24), dtype=torch.int64)
    t[:, 20] = 1 << rank  # different error bits on each rank: the reduce ORs them
    t[:, 13] = 100 + 7 * rank  # makespan max
    t[:, 0] = 5  # a summed field
    t[1, 17] = -(1 << 62)  # the wrapping hash sum (u64 mod 2^64 as int64): 3 * -2^62 wraps to 2^62
    reduce_totals(t, dist)
    if rank == 0:
        out.put(t.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_ors_error_flags_and_maxes_makespan():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_flags_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert list(got[:, 20]) == [7, 7] and list(got[:, 13]) == [114, 114] and list(got[:, 0]) == [15, 15]
    assert got[1, 17] == 1 << 62 and got[0, 17] == 0
