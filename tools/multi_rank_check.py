"""Multi-rank check of the CUDA path (run under torchrun, any world size; gloo on one shared GPU or NCCL on one GPU
per rank): every rank simulates its strong-scaling shard of N config traces with libmig, the per-policy totals are
reduced across ranks (sharding.reduce_totals: one all_gather + sum / max / OR), and rank 0 checks them bit for bit
against one libmig call over all N traces. Prints "MULTI_RANK_OK <world>" on success.
usage: python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/multi_rank_check.py
       [--config 3] [--traces 20000] [--backend gloo]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--traces", type=int, default=20000)
    ap.add_argument("--backend", default="gloo")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2508_18556_b200 as mig
    from paper_2508_18556_b200.sharding import reduce_totals, shard_range
    from tracegen import tracegen as tg

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group(a.backend)
    g = mig.mig_geometry_load(f"builtin:{tg.CONFIG_GEOMETRY[a.config]}")
    specs = [(0, 0), (1, 0), (2, 0), (3, 0), (3, 1), (4, 0)]
    pols = [mig.policy(g, kind=k, flags=f) for k, f in specs]
    seed, J = tg.seed_of(a.config), tg.jobs_per_trace(a.config)
    t0, n = shard_range(rank, world, n_total=a.traces)
    j, e, o = tg.generate_device(a.config, n, trace_id0=t0, seed=seed, device=dev)
    tr = mig.Traces(j, e, o, n, seed=seed, trace_id0=t0, max_jobs=J)
    _, tot = mig.mig_simulate(g, tr, pols)
    t64 = tot.view(torch.int64).view(len(pols), 24)
    reduce_totals(t64, dist)
    torch.cuda.synchronize()
    if rank == 0:
        j, e, o = tg.generate_device(a.config, a.traces, trace_id0=0, seed=seed, device=dev)
        tr = mig.Traces(j, e, o, a.traces, seed=seed, trace_id0=0, max_jobs=J)
        _, ref = mig.mig_simulate(g, tr, pols)
        torch.cuda.synchronize()
        assert torch.equal(ref.view(torch.int64).view(len(pols), 24).cpu(), t64.cpu()), "reduced totals differ"
        assert int(t64[:, 0].sum()) == a.traces * len(pols)
        print(f"MULTI_RANK_OK {world}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
