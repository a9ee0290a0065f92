#!/usr/bin/env python
"""bench.py — MIG-schedule throughput of the B200 hot path (BASELINE.json metric) and its CPU oracle baseline.

A *step* is one pass of the whole hot path over one batch of synthetic traces:
  k_estimate (mig_estimate_memory: per-job memory estimation)
  k_simulate (mig_simulate: tight fit, Alg. 2 placement, fusion/fission, OOM + early restart, event loop,
              per-trace results and per-policy totals, a4-a12)
  [N>1] NCCL all_gather + device reduce of the per-policy totals (the metric reduce of north_star).
Workload at N=1 = BASELINE.json configs[1] (config 2): 10^6 traces x 100 Rodinia-style jobs on A100-40GB under
FUSION_FISSION and BASELINE (the normalisation policy), traces resident in HBM. The same line carries a
`dynamic_path` block: config 4 (10^7 LLM KV-growth traces, FF + early restart), which runs the paper's
dynamic-memory predictor (Alg. 3) and early restart that config 2 does not exercise.

Multi-GPU: weak scaling by default (every rank simulates its own shard of the config's size, trace ids rank*N...);
`--total-traces T` shards T traces over the ranks instead (strong scaling). Shards larger than `--chunk` traces
(config 5: 10^8 traces) are generated on the device chunk by chunk inside the step.

After the timed region the CPU oracle (oracle/, the reported baseline) runs on the host cores over exactly the
trace ids the GPU simulated (all of them when that fits the --cpu-seconds budget, else an evenly strided sample),
compares every covered (trace, policy) row with the device's, and, when it covered the whole launch, the per-policy
totals (decision-hash sum included) bit for bit; the line reports it under "parity".

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference] [--config 2..5]
Under torchrun (N>1) every rank runs; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
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
    5: dict(desc="config5: 100M traces x 50 jobs, A100-40GB, 6-policy sweep, sharded over the GPUs (strong), "
                 "generated on device in chunks of 2^22 traces inside the step",
            traces=100_000_000, total=True, chunk=1 << 22, policies=[(0, 0), (1, 0), (2, 0), (3, 0), (3, 1), (4, 0)]),
}
KIND_OF = {"sim_baseline": 0, "sim_static": 1, "sim_dynamic": 2, "sim_ff": 3, "sim_scheme_a": 4}

# Algorithmic units (SURVEY.md §8(d) "Algorithmic bytes" / "Algorithmic ops"):
OPS_PER_DECISION = 25    # <= 7 legality ANDs + <= 7 fcr lookups + 1 argmax (15-25 integer ops)
OPS_PER_EVENT = 12       # <= 7 compares + queue op + 2 energy ops + 2 hash ops
OPS_PER_DYN_ITER = 23    # RNG + Irwin-Hall ~15, <= 5 level compares, 3 moment updates
OPS_PER_FIT = 25         # per fit until convergence: ~25 FP64 ops incl. 3 divisions and 1 sqrt (+ int128 products)
JOB_BYTES = 16           # job record read once per launch (+16 with an extension record)
RESULT_BYTES = 96        # per-trace result row written once per launch (mig_trace_result)
EST_BYTES = 80           # mig_job_estimate written per DYNAMIC job by k_estimate


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
    """nvidia-smi clocks / throttle reasons sampled every 50 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
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
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def log(msg):
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def _specs(pols):
    return [dict(kind=k, flags=f) for k, f in pols]


# ---------------------------------------------------------------------------------------------------------------
# CPU oracle (the reported baseline and the parity check); test infrastructure, oracle/pool.py
# ---------------------------------------------------------------------------------------------------------------
def oracle_plan(cfg, pols, t_id0, n, procs, budget_s, pool_obj):
    """Calibrate the oracle's cost per trace on a range disjoint from the GPU's ids, then choose the ids it covers:
    all n when that fits budget_s on `procs` processes, else every stride-th id (an even sample)."""
    from oracle import pool

    cal = pool.run(cfg, _specs(pols), t0=t_id0 + n, n=64, procs=1, pool=pool_obj)  # ids after the GPU's range
    per_trace = cal["wall"] / 64
    need_s = n * per_trace / procs
    stride = max(1, math.ceil(need_s / max(budget_s, 1e-3)))
    return stride, per_trace


def oracle_check(cfg, pols, t_id0, n, stride, rows_of, procs, pool_obj, dev_totals=None):
    """Run the oracle over ids t_id0 + k*stride (k = 0..), compare with the device rows rows_of(local ids) element
    by element and, when it covered every trace (stride 1) and dev_totals is given, the per-policy totals."""
    import numpy as np

    from oracle import pool

    local = np.arange(0, n, stride, dtype=np.int64)
    rows = rows_of(None if stride == 1 else local)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "device_rows.npy")
        np.save(path, rows)
        del rows
        if stride == 1:
            r = pool.run(cfg, _specs(pols), t0=t_id0, n=n, procs=procs, cmp_path=path, pool=pool_obj)
        else:
            r = pool.run(cfg, _specs(pols), ids=local + t_id0, procs=procs, cmp_path=path, pool=pool_obj,
                         block=1024)
    totals_equal = None
    if stride == 1 and dev_totals is not None:
        totals_equal = all(int(d[f]) == o[f] for d, o in zip(dev_totals, r["totals"]) for f in pool.TOTALS_FIELDS)
    return r, totals_equal


# ---------------------------------------------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------------------------------------------
class Workload:
    """Device-side inputs of one config shard: resident traces (one mig_simulate per step), or, for shards larger
    than `chunk`, on-device generation of each chunk inside the step (sharding.simulate_generated)."""

    def __init__(self, cfg, n, t_id0, dev, chunk, mig, tg):
        import torch

        self.cfg, self.n, self.t_id0, self.dev, self.mig, self.tg = cfg, n, t_id0, dev, mig, tg
        self.pol_keys = WORKLOADS[cfg]["policies"]
        self.g = mig.mig_geometry_load(f"builtin:{tg.CONFIG_GEOMETRY[cfg]}")
        self.pols = [mig.policy(self.g, kind=k, flags=f) for k, f in self.pol_keys]
        self.n_pol = len(self.pols)
        self.seed = tg.seed_of(cfg)
        self.J = tg.jobs_per_trace(cfg)
        self.chunked = n > chunk
        self.chunk = chunk
        self.stream = torch.cuda.current_stream(dev)
        self.tot = torch.empty((self.n_pol, 192), dtype=torch.uint8, device=dev)
        self.has_ext = tg.has_ext(cfg)
        # the generator's configs without DYNAMIC jobs (config 2) tell the library so: no estimator pass
        self.tflags = 0 if tg.CONFIG_HAS_DYNAMIC[cfg] else mig.MIG_TRACES_NO_DYNAMIC
        if not self.chunked:
            self.jobs, self.ext, self.off = tg.generate_device(cfg, n, trace_id0=t_id0, seed=self.seed, device=dev)
            self.tr = mig.Traces(self.jobs, self.ext, self.off, n, seed=self.seed, trace_id0=t_id0, max_jobs=self.J,
                                 flags=self.tflags)
            self.res = torch.empty((n * self.n_pol, 96), dtype=torch.uint8, device=dev)
            zf = self.jobs[:, 2].to(torch.int64)
            dyn = ((zf >> 16) & 0xFF) == 2
            self.dyn_samples = int(((zf & 0xFFFF) * dyn.to(torch.int64)).sum().item())
            self.n_dyn_jobs = int(dyn.sum().item())
            self.n_jobs = self.tr.n_jobs
            self.fits = self._fits(self.jobs, self.ext, self.off, n, t_id0, zf, dyn) if self.n_dyn_jobs else 0
        else:  # the units the roofline counts, from one pass of the generator over the shard (not timed)
            self.res = None
            self.n_jobs = n * self.J
            self.dyn_samples = self.n_dyn_jobs = self.fits = 0
            for c0 in range(0, n, chunk):
                m = min(chunk, n - c0)
                j, e, o = tg.generate_device(cfg, m, trace_id0=t_id0 + c0, seed=self.seed, device=dev)
                zf = j[:, 2].to(torch.int64)
                dyn = ((zf >> 16) & 0xFF) == 2
                self.dyn_samples += int(((zf & 0xFFFF) * dyn.to(torch.int64)).sum().item())
                self.n_dyn_jobs += int(dyn.sum().item())
                if bool(dyn.any()):
                    self.fits += self._fits(j, e, o, m, t_id0 + c0, zf, dyn)
                del j, e, o, zf, dyn
        self.launches = 0
        self.gen_ms = 0.0

    def _fits(self, jobs, ext, off, n, t_id0, zf, dyn):
        """Fits until convergence (§8(d)) of the shard's DYNAMIC jobs, from one estimator call outside the timed
        region: conv - min_n + 1 for a converged job, T - min_n + 1 otherwise."""
        import torch

        tr = self.mig.Traces(jobs, ext, off, n, seed=self.seed, trace_id0=t_id0, max_jobs=self.J)
        est = self.mig.mig_estimate_memory(self.g, tr, self.pols[0])
        conv = est.view(-1, 80)[:, 8:10].contiguous().view(torch.int16).to(torch.int64).view(-1) & 0xFFFF
        T = zf & 0xFFFF
        min_n = int(self.pols[0].min_n)
        f = torch.where(conv > 0, conv - min_n + 1, (T - min_n + 1).clamp(min=0))
        return int((f * dyn.to(torch.int64)).sum().item())

    def step(self, world, dist):
        import torch

        from paper_2508_18556_b200.sharding import reduce_totals, simulate_generated

        mig = self.mig
        if not self.chunked:
            # one call = the whole hot path: k_estimate (a3 for DYNAMIC jobs; a2 is fused into k_simulate's head
            # evaluation) + k_simulate (a4-a12), per-trace results and per-policy totals in HBM
            mig.mig_simulate(self.g, self.tr, self.pols, est=None, out=self.res, totals=self.tot, stream=self.stream)
            self.launches += mig.mig_last_launch_count()
        else:
            def count(_c0, _m):
                self.launches += mig.mig_last_launch_count()

            red, _ = simulate_generated(self.g, self.cfg, self.pols, self.t_id0, self.n, chunk=self.chunk,
                                        device=self.dev, on_chunk=count)
            self.tot.view(torch.int64).view(self.n_pol, 24).copy_(red)
        if world > 1:  # the per-policy metric reduce over NVLink (NCCL)
            reduce_totals(self.tot.view(torch.int64).view(self.n_pol, 24), dist)

    def rows_of(self, local_ids):
        """Device per-trace results of the shard's local trace ids (None = all) as numpy RESULT_DTYPE rows."""
        import torch

        mig = self.mig
        if self.chunked:  # regenerate the sampled ids' chunks and simulate them with per-trace results
            import numpy as np

            out = []
            ids = np.arange(self.n) if local_ids is None else local_ids
            for c0 in range(0, self.n, self.chunk):
                m = min(self.chunk, self.n - c0)
                sel = ids[(ids >= c0) & (ids < c0 + m)] - c0
                if len(sel) == 0:
                    continue
                t0 = self.t_id0 + c0
                j, e, o = self.tg.generate_device(self.cfg, m, trace_id0=t0, seed=self.seed, device=self.dev)
                tr = mig.Traces(j, e, o, m, seed=self.seed, trace_id0=t0, max_jobs=self.J)
                res, _ = mig.mig_simulate(self.g, tr, self.pols)
                idx = torch.from_numpy(sel).to(self.dev)
                out.append(res.view(m, self.n_pol, 96)[idx].cpu().numpy())
                del j, e, o, tr, res
            return np.concatenate(out).view(mig.RESULT_DTYPE).reshape(-1, self.n_pol)
        res = self.res.view(self.n, self.n_pol, 96)
        if local_ids is not None:
            res = res[torch.from_numpy(local_ids).to(self.dev)]
        return res.cpu().numpy().view(mig.RESULT_DTYPE).reshape(-1, self.n_pol)


def timed(wl, steps, warmup, world, dist, local):
    """W untimed steps, then exactly K steps bracketed by barrier + synchronize, CUDA events on the launching
    stream; per-kernel-group times (mig_timing_enable) and clocks sampled during the timed region."""
    import torch

    mig = wl.mig
    for _ in range(warmup):
        wl.step(world, dist)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wl.launches = 0
    clocks = ClockSampler(local)
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    mig.mig_timing_enable(True)  # CUDA events around each kernel group, on the launching stream
    t_start.record(wl.stream)
    for _ in range(steps):
        wl.step(world, dist)
    t_end.record(wl.stream)
    torch.cuda.synchronize()
    ktimes = mig.mig_timing_query()
    mig.mig_timing_enable(False)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    if world > 1:
        m = torch.tensor([elapsed_ms], device=wl.dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        elapsed_ms = float(m.item())
    return elapsed_ms, ktimes, clk


def roofline(wl, ktimes, steps, totals, world, peaks, peak_src, ncu):
    """Roofline of the dominant kernel (the longest caller-stream launch group per step): algorithmic ops and bytes
    per launch (SURVEY.md §8(d) unit counts x the units one launch processes) / its average CUDA-event duration.
    The bound is chosen by arithmetic intensity against the ridge (ALU peak / HBM peak); both fractions are
    reported."""
    f_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 4 * 32 * f_mhz * 1e6  # lane-ops/s: 4 SMSPs x 1 warp-instruction/cycle x 32 lanes per SM
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
    ridge = alu_peak / hbm_peak
    per_step = {k: v[0] / steps for k, v in ktimes.items()}
    launches = {k: max(1, v[1] // steps) for k, v in ktimes.items()}
    # policies alternate between the caller's stream and a side stream (launch_simulate): a side launch ("~")
    # queues for the SMs of the launch before it, so its event span is not its duration; the dominant launch is
    # taken among the caller-stream launches, whose spans are
    cands = {k: v for k, v in per_step.items() if (k.startswith("sim_") and not k.endswith("~")) or k == "k_estimate"}
    dom = max(cands, key=cands.get)
    n_l = launches[dom]
    ms = per_step[dom] / n_l  # one launch
    ext_b = JOB_BYTES if wl.has_ext else 0
    if dom == "k_estimate":
        # every job record (+ ext) read once, an estimate written per DYNAMIC job; 23 ops per sample scanned
        dyn_samples = wl.dyn_samples or 0
        ops = (OPS_PER_DYN_ITER * dyn_samples + OPS_PER_FIT * (wl.fits or 0)) / n_l
        byts = ((JOB_BYTES + ext_b) * wl.n_jobs + EST_BYTES * (wl.n_dyn_jobs or 0)) / n_l
        ops_desc = (f"{OPS_PER_DYN_ITER} ops per DYNAMIC-job sample scanned + {OPS_PER_FIT} per fit until "
                    f"convergence ({wl.fits} fits)")
        bytes_desc = f"{JOB_BYTES + ext_b} B/job read + {EST_BYTES} B per DYNAMIC job written"
        kname = "k_estimate"
    else:
        # the caller-stream group "sim_<kind>" holds the launches of the policies of that kind with an even index
        # (launch_simulate alternates policy i between the caller's stream, i even, and a side stream)
        even = [i for i, (k, f) in enumerate(wl.pol_keys) if k == KIND_OF[dom] and (i % 2 == 0 or wl.n_pol == 1)]
        dec = sum(int(totals[i]["placements"]) + int(totals[i]["waits"]) + int(totals[i]["rejected"]) for i in even)
        ev = sum(int(totals[i]["placements"]) for i in even)
        # per launch on this rank: the group's decisions / events over its launches (one per policy and chunk)
        ops = (OPS_PER_DECISION * dec + OPS_PER_EVENT * ev) / world / n_l
        byts = ((JOB_BYTES + ext_b) * wl.n_jobs + RESULT_BYTES * wl.n) * len(even) / n_l
        ops_desc = f"{OPS_PER_DECISION}/decision + {OPS_PER_EVENT}/event (SURVEY.md §8(d))"
        bytes_desc = f"{JOB_BYTES + ext_b} B/job read + {RESULT_BYTES} B/trace result written"
        # the fast kernels take extension records and early restart (flag 1), not warp folding / wave time
        fast = all(wl.pol_keys[i][1] in (0, 1) for i in even) and os.environ.get("MIG_FF_FAST", "1") != "0"
        kname = {("sim_ff", True): "k_ff_lane", ("sim_dynamic", True): "k_ff_lane",
                 ("sim_baseline", True): "k_base_lane"}.get((dom, fast), f"k_simulate_lane ({dom})")
    a_ops = ops / (ms * 1e-3)
    a_bytes = byts / (ms * 1e-3)
    intensity = ops / byts if byts else float("inf")
    bound = "hbm" if intensity < ridge else "alu"
    traffic = ncu.get(f"{dom}_dram_bytes_per_launch") if ncu else None
    r = {"bound": bound, "kernel": kname, "ms_per_launch": ms,
         "alu": {"achieved": a_ops, "peak": alu_peak, "unit": "int lane-ops/s", "frac": a_ops / alu_peak,
                 "ops_per_launch": ops, "model": ops_desc,
                 "peak_source": f"148 SMs x 4 SMSP x 32 lanes x {f_mhz:.0f} MHz ({peak_src} sm_max_mhz)"},
         "hbm": {"achieved": a_bytes / 1e9, "peak": hbm_peak / 1e9, "unit": "GB/s", "frac": a_bytes / hbm_peak,
                 "bytes_per_launch": byts, "model": bytes_desc, "peak_source": f"{peak_src} hbm_gbs"},
         "intensity_ops_per_byte": intensity, "ridge_ops_per_byte": ridge}
    if dom != "k_estimate":  # the whole step: every simulation launch's algorithmic units / the step's time
        dec_all = sum(int(t["placements"]) + int(t["waits"]) + int(t["rejected"]) for t in totals) / world
        ev_all = sum(int(t["placements"]) for t in totals) / world
        step_ms = sum(per_step[k] for k in per_step if k == "k_simulate") or ms
        ops_s = OPS_PER_DECISION * dec_all + OPS_PER_EVENT * ev_all
        bytes_s = ((JOB_BYTES + ext_b) * wl.n_jobs + RESULT_BYTES * wl.n) * len(wl.pol_keys)
        r["step"] = {"ms": step_ms, "launches": len(wl.pol_keys), "hbm_frac": bytes_s / (step_ms * 1e-3) / hbm_peak,
                     "alu_frac": ops_s / (step_ms * 1e-3) / alu_peak,
                     "note": "all policy launches of the step (they co-run on two streams) over the k_simulate span"}
    side = r["hbm"] if bound == "hbm" else r["alu"]
    r.update({"achieved": side["achieved"], "peak": side["peak"], "unit": side["unit"], "frac": side["frac"],
              "traffic": traffic})
    if ncu:
        r["ncu_issue_slot_util"] = ncu.get(f"{dom}_issue_slot_util")
        r["ncu_active_lanes_per_instr"] = ncu.get(f"{dom}_active_lanes_per_instr")
        r["ncu_source"] = ncu.get("source")
    return r, dom


def e2e_leg(wl, args, world, dist, dec_step):
    """The same metric end to end through the public C ABI from HOST buffers: every step copies the job records
    host -> device, estimates, simulates and reads the per-policy totals (the metric) back (mig_simulate_host)."""
    import numpy as np
    import torch

    mig = wl.mig
    hj = torch.empty((wl.tr.n_jobs, 4), dtype=torch.int32, pin_memory=True)
    hj.copy_(wl.jobs)
    he = None
    if wl.ext is not None:
        he = torch.empty((wl.tr.n_jobs, 4), dtype=torch.int32, pin_memory=True)
        he.copy_(wl.ext)
    hoff = torch.empty(wl.off.shape, dtype=torch.int64, pin_memory=True)
    hoff.copy_(wl.off)
    ho = hoff.numpy().view("u8")
    hres = torch.empty((wl.n * wl.n_pol, 96), dtype=torch.uint8, pin_memory=True)
    hjn = hj.numpy().view("u4")
    hen = None if he is None else he.numpy().view("u4")
    hresn = hres.numpy().view(mig.RESULT_DTYPE).reshape(wl.n, wl.n_pol)
    htot = np.zeros(wl.n_pol, mig.TOTALS_DTYPE)

    def host_call(with_results):
        mig.mig_simulate_host(wl.g, hjn, hen, ho, wl.pols, seed=wl.seed, trace_id0=wl.t_id0, max_jobs=wl.J,
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
            m = torch.tensor([dt], device=wl.dev)
            dist.all_reduce(m, op=dist.ReduceOp.MAX)
            dt = float(m.item())
        timing[with_results] = dt
    e2e_s = timing[False]
    if world == 1:  # the host path's totals are the device step's, bit for bit
        assert htot.tobytes() == mig.totals_numpy(wl.tot).tobytes(), "e2e totals differ from the device step's"
    h2d = hj.numel() * 4 + (0 if he is None else he.numel() * 4) + ho.nbytes
    d2h = htot.nbytes
    log(f"e2e {e2e_s * 1e3:.1f} ms/step (with per-trace results: {timing[True] * 1e3:.1f})")
    # the PCIe bound of this path: a plain pinned host-to-device copy of the same job records, timed alone
    dj = torch.empty_like(hj, device=wl.dev)
    ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dj.copy_(hj, non_blocking=True)
    ca.record(wl.stream)
    for _ in range(3):
        dj.copy_(hj, non_blocking=True)
    cb.record(wl.stream)
    torch.cuda.synchronize()
    h2d_gbs = 3 * hj.numel() * 4 / (ca.elapsed_time(cb) * 1e-3) / 1e9
    del dj
    return {"value": dec_step / e2e_s, "unit": "decisions/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3, "api": "mig_simulate_host",
            "d2h": "per-policy totals (the metric)",
            "with_per_trace_results": {"ms_per_step": timing[True] * 1e3, "value": dec_step / timing[True],
                                       "d2h_bytes_per_step": int(hres.numel() + htot.nbytes)},
            "pcie_h2d_gbs": h2d_gbs, "h2d_bound_ms": h2d / h2d_gbs / 1e6,
            "frac_of_h2d_bound": (h2d / h2d_gbs / 1e9) / e2e_s}


def load_ncu(cfg, n, full_n):
    prof = os.path.join(ROOT, "profiles", f"ncu_config{cfg}.json")
    if os.path.exists(prof) and n == full_n:
        with open(prof) as f:
            return json.load(f)
    return {}


def measure(cfg, n_per, t_id0, steps, warmup, world, dist, local, dev, chunk, mig, tg, peaks, peak_src):
    """Build the workload, time it, and derive the kernel accounting (one dict, plus the workload object)."""
    wl = Workload(cfg, n_per, t_id0, dev, chunk, mig, tg)
    import torch

    torch.cuda.synchronize()
    log(f"config {cfg}: {n_per} traces (ids {t_id0}..) on {dev}{' in chunks' if wl.chunked else ''}")
    elapsed_ms, ktimes, clk = timed(wl, steps, warmup, world, dist, local)
    totals = mig.totals_numpy(wl.tot)  # all ranks after the reduce
    assert int(totals["error_flags"].max()) == 0, "device reported trace-format errors"
    dec_step = int(sum(int(t["placements"]) + int(t["waits"]) + int(t["rejected"]) for t in totals))
    ms_per_step = elapsed_ms / steps
    full_n = WORKLOADS[cfg]["traces"] // (world if WORKLOADS[cfg].get("total") else 1)
    ncu = load_ncu(cfg, n_per, full_n)
    roof, dom = roofline(wl, ktimes, steps, totals, world, peaks, peak_src, ncu)
    per_step = {k: v[0] / steps for k, v in ktimes.items()}
    m = {"cfg": cfg, "ms_per_step": ms_per_step, "value": dec_step / (ms_per_step * 1e-3), "dec_step": dec_step,
         "traces_per_s": n_per * world / (ms_per_step * 1e-3), "totals": totals, "roofline": roof, "clocks": clk,
         "launches": wl.launches, "kernels": {
             "k_estimate_ms": per_step.get("k_estimate", 0.0), "k_simulate_ms": per_step.get("k_simulate", 0.0),
             "launch_ms": {k: v for k, v in per_step.items() if k not in ("k_estimate", "k_simulate")},
             "dominant": dom, "dominant_share": per_step[dom] / ms_per_step}}
    if wl.dyn_samples:  # §8(d): configs 3-4 are dominated by predictor steps
        m["iteration_steps_per_s"] = wl.dyn_samples * world / (ms_per_step * 1e-3)
    return m, wl


def cpu_leg(wl, m, args, world, procs, pool_obj, budget_s):
    """The oracle over the rank's GPU ids (all, or an even sample within the budget): cpu_baseline + parity."""
    dev_tot = m["totals"] if world == 1 else None
    stride, per_trace = oracle_plan(wl.cfg, wl.pol_keys, wl.t_id0, wl.n, procs, budget_s, pool_obj)
    r, totals_equal = oracle_check(wl.cfg, wl.pol_keys, wl.t_id0, wl.n, stride, wl.rows_of, procs, pool_obj,
                                   dev_totals=dev_tot)
    ids = (f"all {wl.n} trace ids {wl.t_id0}..{wl.t_id0 + wl.n - 1}" if stride == 1 else
           f"{r['traces']} trace ids {wl.t_id0}, {wl.t_id0 + stride}, ... (every {stride}th of the GPU's "
           f"{wl.n})")
    sample = f"{ids} of config {wl.cfg} x {len(wl.pol_keys)} policies, {r['procs']} processes"
    cpu = {"value": r["decisions"] / r["wall"], "unit": "decisions/s", "cores": r["procs"], "kind": "oracle",
           "sample": sample, "traces_per_s": r["traces"] / r["wall"], "wall_s": round(r["wall"], 2),
           "per_process_decisions_per_s": r["per_process_decisions_per_s"], "cpu_model": cpu_model(),
           "host_cpus": os.cpu_count()}
    parity = {"mode": "full" if stride == 1 else f"sampled (every {stride}th trace)", "traces_checked": r["traces"],
              "rows_checked": r["traces"] * len(wl.pol_keys), "rows_mismatched": r["mismatches"],
              "first_mismatch": r["first"], "totals_equal": totals_equal,
              "rule": "every integer field and the decision hash of every (trace, policy) row bit-exact; "
                      "per-policy totals (decision_hash_sum included) bit-exact when every trace is covered"}
    log(f"oracle over {r['traces']} traces: {r['mismatches']} mismatched rows, totals_equal={totals_equal}")
    return cpu, parity


def run_mine(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = args.config
    spec = WORKLOADS[cfg]
    from paper_2508_18556_b200.sharding import shard_range

    total = args.total_traces or (spec["traces"] if spec.get("total") and not args.traces else 0)
    if total:
        t_id0, n_per = shard_range(rank, world, n_total=total)
        scaling = "strong"
    else:
        n_per = args.traces or spec["traces"]
        t_id0, _ = shard_range(rank, world, n_per_rank=n_per)
        scaling = "weak"

    local = local % max(1, torch.cuda.device_count())  # --share-gpu testing: several ranks on one device
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # functional test of the multi-rank path on a single-GPU box (NCCL refuses a shared device)
            dist.init_process_group(args.dist_backend)
    import paper_2508_18556_b200 as mig
    from tracegen import tracegen as tg

    peaks, peak_src = measured_peaks()
    chunk = args.chunk or spec.get("chunk", 1 << 62)
    m, wl = measure(cfg, n_per, t_id0, args.steps, args.warmup, world, dist, local, dev, chunk, mig, tg, peaks,
                    peak_src)
    log(f"timed {args.steps} steps: {m['ms_per_step']:.3f} ms/step")
    e2e = None
    if not args.no_e2e and not wl.chunked:
        e2e = e2e_leg(wl, args, world, dist, m["dec_step"])
    elif not args.no_e2e:
        e2e = {"value": None, "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": "chunked shard: inputs are generated on the device inside the step; no host-buffer leg"}

    # the paper's dynamic-memory path (Alg. 3 predictor + early restart) in the same run: config 4
    dyn = None
    if cfg == 2 and not args.no_dynamic:
        n4 = args.dynamic_traces or WORKLOADS[4]["traces"]
        t4, _ = shard_range(rank, world, n_per_rank=n4)
        m4, wl4 = measure(4, n4, t4, args.dynamic_steps, max(3, min(args.warmup, 3)), world, dist, local, dev,
                          args.chunk or (1 << 62), mig, tg, peaks, peak_src)
        dyn = {"workload": WORKLOADS[4]["desc"], "traces_per_gpu": n4, "jobs_per_trace": wl4.J,
               "policies": [POLICY_NAMES[p] for p in wl4.pol_keys], "steps": args.dynamic_steps,
               "warmup": max(3, min(args.warmup, 3)), "ms_per_step": m4["ms_per_step"],
               "value": m4["value"], "unit": "decisions/s", "traces_per_s": m4["traces_per_s"],
               "iteration_steps_per_s": m4.get("iteration_steps_per_s"),
               "dynamic_samples_per_step": wl4.dyn_samples, "decisions_per_step": m4["dec_step"],
               "early_restart": {"preempts": int(m4["totals"][0]["preempts"]), "ooms_ff_er": int(m4["totals"][0]["ooms"]),
                                 "ooms_ff": int(m4["totals"][1]["ooms"]),
                                 "wasted_ticks_ff_er": int(m4["totals"][0]["wasted_ticks"]),
                                 "wasted_ticks_ff": int(m4["totals"][1]["wasted_ticks"])},
               "kernels": m4["kernels"], "roofline": m4["roofline"], "clocks": m4["clocks"],
               "gpu_launches": m4["launches"]}
        m["launches_dynamic"] = m4["launches"]
        log(f"dynamic path (config 4): {m4['ms_per_step']:.2f} ms/step")

    # the CPU oracle on the host cores, after the timed regions: baseline rate + parity over the GPU's ids
    cpu = parity = None
    if rank == 0 and not args.no_cpu:
        import multiprocessing as mp

        procs = min(os.cpu_count() or 1, args.cpu_cores)
        pool_obj = mp.get_context("spawn").Pool(procs)
        try:
            cpu, parity = cpu_leg(wl, m, args, world, procs, pool_obj, args.cpu_seconds)
            if dyn is not None:
                c4, p4 = cpu_leg(wl4, m4, args, world, procs, pool_obj, args.cpu_seconds_dynamic)
                dyn["cpu_baseline"] = c4
                dyn["parity"] = p4
        finally:
            pool_obj.close()
            pool_obj.join()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": m["value"], "unit": "decisions/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "int32/int64 (+f64 predictor)",
        "data": "synthetic (seeded counter-based tracegen, generated on device)",
        "traces_per_s": m["traces_per_s"],
        "config": {"workload": spec["desc"], "traces_per_gpu": n_per, "total_traces": n_per * world if not total
                   else total, "jobs_per_trace": wl.J, "policies": [POLICY_NAMES[p] for p in wl.pol_keys],
                   "decisions_per_step": m["dec_step"],
                   "decisions_by_policy": {POLICY_NAMES[p]: int(t["placements"]) + int(t["waits"]) + int(t["rejected"])
                                           for p, t in zip(wl.pol_keys, m["totals"])},
                   "parallelism": f"trace-sharded x{world} ({scaling})",
                   "l2": (f"inputs ({wl.n_jobs * 16 / 1e9:.2f} GB/GPU) larger than L2; no flush" if not wl.chunked
                          else "inputs generated per chunk inside the step (chunks larger than L2); no flush")},
        "kernels": m["kernels"],
        "roofline": m["roofline"],
        "parity": parity,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": m["launches"],
        "clocks": m["clocks"],
        "dynamic_path": dyn,
    }
    if "iteration_steps_per_s" in m:
        line["iteration_steps_per_s"] = m["iteration_steps_per_s"]
    print(json.dumps(line), flush=True)
    if parity and parity["rows_mismatched"]:
        print(f"PARITY FAILURE: {parity['first_mismatch']}", file=sys.stderr)
    if world > 1:
        dist.destroy_process_group()
    if (parity and (parity["rows_mismatched"] or parity["totals_equal"] is False)) or \
            (dyn and dyn.get("parity") and dyn["parity"]["rows_mismatched"]):
        sys.exit(3)


def run_reference(args):
    """The reference arm of this tier: the CPU oracle as it stands, timed on the host cores over bounded samples
    of the same workload; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp

    from oracle import pool

    spec = WORKLOADS[args.config]
    procs = min(os.cpu_count() or 1, args.cpu_cores)
    pool_obj = mp.get_context("spawn").Pool(procs)
    rates, trates, walls = [], [], []
    sample = ""
    try:
        cal = pool.run(args.config, _specs(spec["policies"]), t0=0, n=16, procs=1, pool=pool_obj)
        per_proc = max(procs, int(args.ref_seconds / max(cal["wall"] / 16, 1e-6)))
        n = per_proc * procs
        for step in range(args.warmup + args.steps):
            t0 = step * n
            r = pool.run(args.config, _specs(spec["policies"]), t0=t0, n=n, procs=procs, pool=pool_obj)
            sample = f"{n} traces of config {args.config} (ids {t0}..{t0 + n - 1}), {procs} processes"
            if step >= args.warmup:
                rates.append(r["decisions"] / r["wall"])
                trates.append(r["traces"] / r["wall"])
                walls.append(r["wall"])
    finally:
        pool_obj.close()
        pool_obj.join()
    value = sum(rates) / len(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "decisions/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32/int64 (+f64 predictor)",
        "data": "synthetic (seeded tracegen)", "traces_per_s": sum(trates) / len(trates),
        "config": {"workload": spec["desc"], "policies": [POLICY_NAMES[p] for p in spec["policies"]],
                   "parallelism": f"{procs} oracle processes"},
        "cpu_baseline": {"value": value, "unit": "decisions/s", "cores": procs, "kind": "oracle",
                         "sample": f"per step: {sample}", "cpu_model": cpu_model(), "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["mine", "reference"], default="mine")
    ap.add_argument("--config", type=int, default=2, choices=sorted(WORKLOADS))
    ap.add_argument("--traces", type=int, default=0, help="traces per GPU (weak scaling; default: the config's)")
    ap.add_argument("--total-traces", type=int, default=0, help="traces over all GPUs (strong scaling)")
    ap.add_argument("--chunk", type=int, default=0,
                    help="shards larger than this are generated in chunks (default: 2^22 for config 5, else none)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dynamic", action="store_true", help="skip the config-4 dynamic_path block")
    ap.add_argument("--dynamic-traces", type=int, default=0)
    ap.add_argument("--dynamic-steps", type=int, default=5)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="oracle budget (s) for the main workload")
    ap.add_argument("--cpu-seconds-dynamic", type=float, default=10.0)
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
