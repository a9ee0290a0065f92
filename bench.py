#!/usr/bin/env python
"""bench.py — MIG-schedule throughput of the B200 hot path (BASELINE.json metric) and its CPU oracle baseline.

A *step* is one pass of the whole hot path over one batch of device-resident synthetic traces:
  k_estimate (mig_estimate_memory: per-job memory estimation)
  k_simulate (mig_simulate: tight fit, Alg. 2 placement, fusion/fission, OOM + early restart, event loop,
              per-trace results and per-policy totals, a4-a12)
  [N>1] NCCL all_gather + device reduce of the per-policy totals (the metric reduce of north_star).
Workload at N=1 = BASELINE.json configs[1] (config 2): 10^6 traces x 100 Rodinia-style jobs on A100-40GB under
FUSION_FISSION and BASELINE (the normalisation policy). Multi-GPU is weak scaling: every rank simulates its own
10^6-trace shard (trace ids rank*N ...), no data-path collective, one metric all_gather per step.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference] [--config 2..5]
Under torchrun (N>1) every rank runs; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

with open(os.path.join(ROOT, "BASELINE.json")) as _f:
    METRIC = json.load(_f)["metric"]

POLICY_NAMES = {(0, 0): "BASELINE", (1, 0): "STATIC", (2, 0): "DYNAMIC", (3, 0): "FUSION_FISSION",
                (3, 1): "FUSION_FISSION|EARLY_RESTART", (4, 0): "SCHEME_A", (4, 1): "SCHEME_A|EARLY_RESTART"}
WORKLOADS = {
    2: dict(desc="config2: 1M Monte-Carlo traces x 100 Rodinia-style jobs, A100-40GB, FUSION_FISSION (+BASELINE)",
            traces=1_000_000, policies=[(3, 0), (0, 0)]),
    3: dict(desc="config3: 1M traces x 20 ML jobs (25% dynamic), A100-80GB, FF+EARLY_RESTART (+FF, BASELINE)",
            traces=1_000_000, policies=[(3, 1), (3, 0), (0, 0)]),
    4: dict(desc="config4: 10M LLM KV-growth traces x 4 jobs, H100-80GB, FF+EARLY_RESTART (+FF, BASELINE)",
            traces=10_000_000, policies=[(3, 1), (3, 0), (0, 0)]),
    5: dict(desc="config5 (per-GPU shard of 100M): 12.5M traces x 50 jobs, A100-40GB, 6-policy sweep",
            traces=12_500_000, policies=[(0, 0), (1, 0), (2, 0), (3, 0), (3, 1), (4, 0)]),
}

# Algorithmic integer-op model of the hot path: lane-ops an ideal scalar implementation
# of the method's definitions needs per unit, on an 8-slot geometry.
OPS_PER_DECISION = 64   # head evaluation: tight fit, reuse scan over <=7 slices, Alg. 2 over <=7 placements, record
OPS_PER_EVENT = 24      # next event over <=7 running slices, apply, record, energy
OPS_PER_JOB_STAGE = 10  # per job and policy: load, tight fit, stage
OPS_PER_DYN_ITER = 24   # per dynamic-job sample scanned: counter RNG, Irwin-Hall, level checks, moment update


def _oracle_worker(args):
    cfg, t0, n, pols, seconds_hint = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import oracle as orc
    from tracegen import tracegen as tg

    jobs, ext, off = tg.generate_host(cfg, n, trace_id0=t0)
    g = orc.Geometry(os.path.join(ROOT, "paper_2508_18556_b200", "geometries", tg.CONFIG_GEOMETRY[cfg] + ".json"))
    opols = [orc.policy(kind=k, flags=f) for k, f in pols]
    t = time.perf_counter()
    r = orc.simulate(g, jobs, ext, off, opols, seed=tg.seed_of(cfg), trace_id0=t0)
    dt = time.perf_counter() - t
    dec = int(r["placements"].astype("u8").sum() + r["waits"].astype("u8").sum() + r["rejected"].astype("u8").sum())
    return dt, dec, n


def oracle_rate(cfg, pols, cores, seconds, first_trace=0, pool=None, max_traces=0):
    """Time the CPU oracle (as it stands, single-threaded per process) on `cores` processes over a bounded sample
    of the workload sized for ~`seconds` of CPU work per process. Returns (decisions/s, traces/s, sample desc)."""
    import multiprocessing as mp

    own = pool is None
    if own:
        pool = mp.get_context("spawn").Pool(cores)  # fresh interpreters: no fork after OpenMP / CUDA init
    try:
        # calibrate on a small run in a worker
        dt, dec, n = pool.apply(_oracle_worker, ((cfg, first_trace, 64, pols, 0),))
        per_core = max(16, int(64 * seconds / max(dt, 1e-6)))
        if max_traces:
            per_core = max(16, min(per_core, max_traces // cores))  # never more than the workload itself
        tasks = [(cfg, first_trace + 64 + i * per_core, per_core, pols, seconds) for i in range(cores)]
        outs = pool.map_async(_oracle_worker, tasks).get(timeout=max(120.0, 20 * seconds))
    finally:
        if own:
            pool.close()
            pool.join()
    wall = max(o[0] for o in outs)
    decs = sum(o[1] for o in outs)
    ntr = sum(o[2] for o in outs)
    sample = (f"{ntr} traces of config {cfg} (ids {first_trace + 64}..{first_trace + 64 + ntr - 1}) x "
              f"{len(pols)} policies, {cores} processes x {per_core} traces")
    oracle_rate.single = statistics.mean(o[1] / o[0] for o in outs)  # one process (one core) alone
    return decs / wall, ntr / wall, sample, wall


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def run_reference(args):
    """The reference arm of this tier: the CPU oracle timed on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = WORKLOADS[args.config]
    cores = min(os.cpu_count() or 1, args.cpu_cores)
    import multiprocessing as mp

    pool = mp.get_context("spawn").Pool(cores)
    rates, trates, walls = [], [], []
    sample = ""
    try:
        for step in range(args.warmup + args.steps):
            r, tr, sample, wall = oracle_rate(args.config, wl["policies"], cores, args.ref_seconds,
                                              first_trace=step * 1_000_000, pool=pool)
            if step >= args.warmup:
                rates.append(r)
                trates.append(tr)
                walls.append(wall)
    finally:
        pool.close()
        pool.join()
    value = sum(rates) / len(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "decisions/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32/int64 (+f64 predictor)",
        "data": "synthetic (seeded tracegen)", "traces_per_s": sum(trates) / len(trates),
        "config": {"workload": wl["desc"], "policies": [POLICY_NAMES[p] for p in wl["policies"]],
                   "parallelism": f"{cores} oracle processes"},
        "cpu_baseline": {"value": value, "unit": "decisions/s", "cores": cores, "kind": "oracle",
                         "sample": f"per step: {sample}", "cpu_model": cpu_model(), "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def log(msg):
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def run_mine(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    wl = WORKLOADS[args.config]
    n_per = args.traces or wl["traces"]
    cfg = args.config

    # CPU oracle baseline first (rank 0, N=1), before CUDA is initialised (forked workers).
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = min(os.cpu_count() or 1, args.cpu_cores)
        r, trs, sample, wall = oracle_rate(cfg, wl["policies"], cores, args.cpu_seconds, max_traces=n_per)
        cpu = {"value": r, "unit": "decisions/s", "cores": cores, "kind": "oracle", "sample": sample,
               "traces_per_s": trs, "wall_s": round(wall, 2), "per_process_decisions_per_s": oracle_rate.single,
               "cpu_model": cpu_model(), "host_cpus": os.cpu_count()}
        log(f"cpu oracle baseline: {r:.3e} decisions/s on {cores} cores")

    local = local % max(1, torch.cuda.device_count())  # --share-gpu testing: several ranks on one device
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # functional test of the multi-rank path on a single-GPU box (NCCL refuses a shared device)
            dist.init_process_group(args.dist_backend)
    import paper_2508_18556_b200 as mig
    from paper_2508_18556_b200.sharding import reduce_totals, shard_range
    from tracegen import tracegen as tg

    stream = torch.cuda.current_stream(dev)
    g = mig.mig_geometry_load(f"builtin:{tg.CONFIG_GEOMETRY[cfg]}")
    pols = [mig.policy(g, kind=k, flags=f) for k, f in wl["policies"]]
    n_pol = len(pols)
    seed = tg.seed_of(cfg)
    t_id0, _ = shard_range(rank, world, n_per_rank=n_per)
    jobs, ext, off = tg.generate_device(cfg, n_per, trace_id0=t_id0, seed=seed, device=dev)
    J = tg.jobs_per_trace(cfg)
    # samples the estimator scans per step (a3 runs every DYNAMIC job to its declared T): iteration-steps (§8(d))
    zf = jobs[:, 2].to(torch.int64)
    dyn_samples = int(((zf & 0xFFFF) * (((zf >> 16) & 0xFF) == 2).to(torch.int64)).sum().item())
    tr = mig.Traces(jobs, ext, off, n_per, seed=seed, trace_id0=t_id0, max_jobs=J)
    res = torch.empty((n_per * n_pol, 96), dtype=torch.uint8, device=dev)
    tot = torch.empty((n_pol, 192), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    log(f"generated {n_per} traces of config {cfg} on {dev}")

    launches = 0

    def step():
        # one call = the whole hot path: k_estimate (a3 for DYNAMIC jobs; a2 is fused into k_simulate's head
        # evaluation) + k_simulate (a4-a12), per-trace results and per-policy totals in HBM
        nonlocal launches
        mig.mig_simulate(g, tr, pols, est=None, out=res, totals=tot, stream=stream)
        launches += mig.mig_last_launch_count()
        if world > 1:  # the per-policy metric reduce over NVLink (NCCL)
            reduce_totals(tot.view(torch.int64).view(n_pol, 24), dist)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    log("warm-up done")
    if world > 1:
        dist.barrier()
    launches = 0
    clocks = ClockSampler(local)
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    mig.mig_timing_enable(True)  # CUDA events around each kernel group, on the launching stream
    t_start.record(stream)
    for k in range(args.steps):
        step()
    t_end.record(stream)
    torch.cuda.synchronize()
    ktimes = mig.mig_timing_query()
    mig.mig_timing_enable(False)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    log(f"timed {args.steps} steps: {t_start.elapsed_time(t_end):.1f} ms")
    elapsed_ms = t_start.elapsed_time(t_end)
    est_ms = ktimes.get("k_estimate", (0.0, 0))[0] / args.steps
    sim_ms = ktimes.get("k_simulate", (0.0, 0))[0] / args.steps
    if world > 1:
        m = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        elapsed_ms = float(m.item())
    totals = mig.totals_numpy(tot)  # all ranks after the reduce
    assert int(totals["error_flags"].max()) == 0, "device reported trace-format errors"
    dec_step = int(sum(int(t["placements"]) + int(t["waits"]) + int(t["rejected"]) for t in totals))
    events_step = int(sum(int(t["placements"]) for t in totals))
    jobs_step = int(totals[0]["n_jobs"])
    ms_per_step = elapsed_ms / args.steps
    value = dec_step / (ms_per_step * 1e-3)
    traces_per_s = n_per * world / (ms_per_step * 1e-3)

    # ---- end to end through the public C ABI from HOST buffers (H2D + estimate + simulate + D2H per step) ----
    e2e = None
    if not args.no_e2e:
        hj = torch.empty((tr.n_jobs, 4), dtype=torch.int32, pin_memory=True)
        hj.copy_(jobs)
        he = None
        if ext is not None:
            he = torch.empty((tr.n_jobs, 4), dtype=torch.int32, pin_memory=True)
            he.copy_(ext)
        hoff = torch.empty(off.shape, dtype=torch.int64, pin_memory=True)
        hoff.copy_(off)
        ho = hoff.numpy().view("u8")
        hres = torch.empty((n_per * n_pol, 96), dtype=torch.uint8, pin_memory=True)
        hjn = hj.numpy().view("u4")
        hen = None if he is None else he.numpy().view("u4")
        hresn = hres.numpy().view(mig.RESULT_DTYPE).reshape(n_per, n_pol)
        import numpy as np

        htot = np.zeros(n_pol, mig.TOTALS_DTYPE)

        def host_call(with_results):
            mig.mig_simulate_host(g, hjn, hen, ho, pols, seed=seed, trace_id0=t_id0, max_jobs=J,
                                  out=hresn if with_results else None, totals=htot, results=with_results)

        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        timing = {}
        for with_results in (False, True):  # the metric (per-policy totals) back; then also every per-trace result
            for _ in range(2):  # warm-up calls (first-call host allocations and page mapping)
                host_call(with_results)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                host_call(with_results)
            dt = (time.perf_counter() - t0) / e2e_steps
            if world > 1:
                m = torch.tensor([dt], device=dev)
                dist.all_reduce(m, op=dist.ReduceOp.MAX)
                dt = float(m.item())
            timing[with_results] = dt
        e2e_s = timing[False]
        if world == 1:  # the host path's totals are the device step's, bit for bit
            assert htot.tobytes() == mig.totals_numpy(tot).tobytes(), "e2e totals differ from the device step's"
        h2d = hj.numel() * 4 + (0 if he is None else he.numel() * 4) + ho.nbytes
        d2h = htot.nbytes
        log(f"e2e {e2e_s * 1e3:.1f} ms/step (with per-trace results: {timing[True] * 1e3:.1f})")
        # the PCIe bound of this path: a plain pinned host-to-device copy of the same job records, timed alone
        dj = torch.empty_like(hj, device=dev)
        ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dj.copy_(hj, non_blocking=True)
        ca.record(stream)
        for _ in range(3):
            dj.copy_(hj, non_blocking=True)
        cb.record(stream)
        torch.cuda.synchronize()
        h2d_gbs = 3 * hj.numel() * 4 / (ca.elapsed_time(cb) * 1e-3) / 1e9
        del dj
        e2e = {"value": dec_step / e2e_s, "unit": "decisions/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3, "api": "mig_simulate_host",
               "d2h": "per-policy totals (the metric)",
               "with_per_trace_results": {"ms_per_step": timing[True] * 1e3, "value": dec_step / timing[True],
                                          "d2h_bytes_per_step": int(hres.numel() + htot.nbytes)},
               "pcie_h2d_gbs": h2d_gbs, "h2d_bound_ms": h2d / h2d_gbs / 1e6,
               "frac_of_h2d_bound": (h2d / h2d_gbs / 1e9) / e2e_s}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks, peak_src = measured_peaks()
    f_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 4 * 32 * f_mhz * 1e6  # lane-ops/s: 4 SMSPs x 1 warp-instruction/cycle x 32 lanes per SM
    # Roofline of the dominant launch (the longest per-policy simulation launch, timed by CUDA events on the
    # launching stream through mig_timing_enable): algorithmic lane-ops of that policy's decisions and events
    # (DESIGN.md ops model) / its average launch duration, against the issue peak.
    launch_ms = {k: v[0] / args.steps for k, v in ktimes.items() if k.startswith("sim_")}
    # policies alternate between the caller's stream and a side stream (launch_simulate): a side launch ("~")
    # queues for the SMs of the launch before it, so its event span is not its duration; the dominant launch is
    # taken among the caller-stream launches, whose spans are
    own = {k: v for k, v in launch_ms.items() if not k.endswith("~")}
    dom = max(own, key=own.get) if own else "k_simulate"
    dom_ms = launch_ms.get(dom, sim_ms)
    kind_of = {"sim_baseline": 0, "sim_static": 1, "sim_dynamic": 2, "sim_ff": 3}
    dom_pols = [i for i, (k, f) in enumerate(wl["policies"]) if k == kind_of.get(dom, -1)] or list(range(n_pol))
    dom_dec = sum(int(totals[i]["placements"]) + int(totals[i]["waits"]) + int(totals[i]["rejected"]) for i in dom_pols)
    dom_ev = sum(int(totals[i]["placements"]) for i in dom_pols)
    dom_launches = max(1, ktimes.get(dom, (0, args.steps))[1] // args.steps) if dom in ktimes else 1
    ops_dom = (OPS_PER_DECISION * dom_dec + OPS_PER_EVENT * dom_ev +
               OPS_PER_JOB_STAGE * jobs_step * len(dom_pols)) / world / dom_launches
    achieved = ops_dom / (dom_ms / dom_launches * 1e-3)
    ops_desc = f"{OPS_PER_DECISION}/decision + {OPS_PER_EVENT}/event + {OPS_PER_JOB_STAGE}/job/policy (DESIGN.md)"
    kname = f"k_simulate_lane ({dom})"
    if est_ms > dom_ms and dyn_samples:  # configs 3-4: the estimator is the dominant kernel (one launch per step)
        dom, dom_ms, kname, dom_launches = "k_estimate", est_ms, "k_estimate", 1
        achieved = OPS_PER_DYN_ITER * dyn_samples / (est_ms * 1e-3)
        ops_desc = f"{OPS_PER_DYN_ITER}/DYNAMIC-job sample scanned (fits not counted; DESIGN.md)"
    traffic, ncu = None, {}
    prof = os.path.join(ROOT, "profiles", f"ncu_config{cfg}.json")
    if os.path.exists(prof) and n_per == wl["traces"]:
        with open(prof) as f:
            ncu = json.load(f)
        traffic = ncu.get(f"{dom}_dram_bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": "decisions/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32/int64 (+f64 predictor)",
        "data": "synthetic (seeded counter-based tracegen, generated on device)",
        "traces_per_s": traces_per_s,
        "config": {"workload": wl["desc"], "traces_per_gpu": n_per, "jobs_per_trace": J,
                   "policies": [POLICY_NAMES[p] for p in wl["policies"]],
                   "decisions_per_step": dec_step, "parallelism": f"trace-sharded x{world}",
                   "l2": f"inputs ({tr.n_jobs * 16 / 1e9:.2f} GB/GPU) larger than L2; no flush"},
        "kernels": {"k_estimate_ms": est_ms, "k_simulate_ms": sim_ms,
                    "k_simulate_share": sim_ms / ms_per_step, "launch_ms": launch_ms,
                    "dominant_share": dom_ms / ms_per_step},
        "roofline": {"bound": "alu", "kernel": kname, "achieved": achieved, "peak": alu_peak,
                     "unit": "int lane-ops/s", "frac": achieved / alu_peak, "traffic": traffic,
                     "peak_source": f"148 SMs x 4 SMSP x 32 lanes x {f_mhz:.0f} MHz ({peak_src} sm_max_mhz)",
                     "ops_model": ops_desc,
                     "ncu_issue_slot_util": ncu.get(f"{dom}_issue_slot_util"),
                     "ncu_active_lanes_per_instr": ncu.get(f"{dom}_active_lanes_per_instr"),
                     "ncu_source": ncu.get("source")},
        # secondary roofline: a launch reads every job record once and writes one 96 B result per trace
        "hbm": {"algorithmic_bytes_per_launch": tr.n_jobs * 16 + n_per * 96, "peak_gbs": peaks.get("hbm_gbs")},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
    }
    line["hbm"]["achieved_gbs"] = line["hbm"]["algorithmic_bytes_per_launch"] / (dom_ms / dom_launches * 1e-3) / 1e9
    if dyn_samples:  # §8(d): configs 3-4 are dominated by predictor steps
        line["iteration_steps_per_s"] = dyn_samples * world / (ms_per_step * 1e-3)
        line["config"]["dynamic_samples_per_step"] = dyn_samples
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["mine", "reference"], default="mine")
    ap.add_argument("--config", type=int, default=2, choices=sorted(WORKLOADS))
    ap.add_argument("--traces", type=int, default=0, help="traces per GPU (default: the config's)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-cores", type=int, default=64)
    ap.add_argument("--ref-seconds", type=float, default=2.0)
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default) or gloo (multi-rank test on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
