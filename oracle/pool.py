"""Multi-process runner of the CPU oracle over a trace-id set. TEST INFRASTRUCTURE ONLY.

Only tests/ and bench.py's cpu_baseline / ``--impl reference`` legs use this module. Each worker process
regenerates its traces on the host (tracegen, the shared input generator) and runs the single-threaded oracle
(oracle.cpp) on them; nothing here touches the CUDA path. Optionally a worker compares its oracle results, element
by element, with a results file written by the caller (the device's per-trace results, RESULT_DTYPE rows), so that
10^6-trace parity checks never move the oracle's results between processes.

Per-policy totals are formed from the oracle's per-trace results by their plain definitions (sums over traces,
wrapping mod 2^64 for the decision-hash sum, the maximum makespan), in the mig_policy_totals field order.
"""
from __future__ import annotations

import os
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M64 = (1 << 64) - 1

TOTALS_FIELDS = ["n_traces", "n_jobs", "completed", "rejected", "failed", "ooms", "preempts", "restarts",
                 "placements", "waits", "creates", "destroys", "makespan_sum", "makespan_max", "energy_wticks",
                 "turnaround_sum", "busy_slice_ticks", "decision_hash_sum", "mem_mib_ticks", "wasted_ticks",
                 "error_flags", "reserved0", "reserved1", "reserved2"]
_SUMMED = {"n_jobs": "n_jobs", "completed": "completed", "rejected": "rejected", "failed": "failed",
           "ooms": "ooms", "preempts": "preempts", "restarts": "restarts", "placements": "placements",
           "waits": "waits", "creates": "creates", "destroys": "destroys", "makespan_sum": "makespan",
           "energy_wticks": "energy_wticks", "turnaround_sum": "turnaround_sum",
           "busy_slice_ticks": "busy_slice_ticks", "decision_hash_sum": "decision_hash",
           "mem_mib_ticks": "mem_mib_ticks", "wasted_ticks": "wasted_ticks"}


def totals_of(res):
    """Per-policy totals (list of dicts, python ints) of oracle results res[n_traces, n_pol]."""
    out = []
    for p in range(res.shape[1]):
        r = res[:, p]
        t = {f: 0 for f in TOTALS_FIELDS}
        t["n_traces"] = len(r)
        for f, src in _SUMMED.items():
            t[f] = int(r[src].astype(np.uint64).sum(dtype=np.uint64)) & M64
        t["makespan_max"] = int(r["makespan"].max(initial=0))
        out.append(t)
    return out


def merge_totals(parts):
    """Combine per-worker totals: sums wrap mod 2^64, makespan_max is a maximum, error_flags an OR."""
    if not parts:
        return []
    out = [dict(t) for t in parts[0]]
    for part in parts[1:]:
        for o, t in zip(out, part):
            for f in TOTALS_FIELDS:
                if f == "makespan_max":
                    o[f] = max(o[f], t[f])
                elif f == "error_flags":
                    o[f] |= t[f]
                else:
                    o[f] = (o[f] + t[f]) & M64
    return out


def _geometry(cfg):
    from oracle import oracle as orc
    from tracegen import tracegen as tg

    return orc.Geometry(os.path.join(ROOT, "paper_2508_18556_b200", "geometries", tg.CONFIG_GEOMETRY[cfg] + ".json"))


def _first_mismatch(got, want):
    for f in want.dtype.names:
        if not np.array_equal(got[f], want[f]):
            k = tuple(np.argwhere(got[f] != want[f])[0])
            return f, k, int(got[f][k]), int(want[f][k])
    return None


def _work(args):
    """One worker: traces `ids` (an int64 array of trace ids) or the range [t0, t0 + n) of config cfg under specs.
    Returns timing, decision count, per-policy totals, and the comparison against cmp_path rows [row0, ...)."""
    cfg, t0, n, ids, specs, block, cmp_path, row0, want_results = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import oracle as orc
    from tracegen import tracegen as tg

    seed = tg.seed_of(cfg)
    g = _geometry(cfg)
    opols = [orc.policy(**s) for s in specs]
    cmp = np.load(cmp_path, mmap_mode="r") if cmp_path else None
    sim_s = 0.0
    parts, results = [], []
    bad, first = 0, None
    count = len(ids) if ids is not None else n
    k = 0
    while k < count:
        if ids is None:  # contiguous ids: one generator call and one oracle call per block
            m = min(block, count - k)
            jobs, ext, off = tg.generate_host(cfg, m, trace_id0=t0 + k)
            t = time.perf_counter()
            r = orc.simulate(g, jobs, ext, off, opols, seed=seed, trace_id0=t0 + k)
            sim_s += time.perf_counter() - t
        else:  # arbitrary ids (strided samples): one trace per call
            m = min(block, count - k)
            r = np.zeros((m, len(opols)), orc.RESULT_DTYPE)
            for i in range(m):
                tid = int(ids[k + i])
                jobs, ext, off = tg.generate_host(cfg, 1, trace_id0=tid)
                t = time.perf_counter()
                r[i] = orc.simulate(g, jobs, ext, off, opols, seed=seed, trace_id0=tid)[0]
                sim_s += time.perf_counter() - t
        parts.append(totals_of(r))
        if cmp is not None:
            got = np.asarray(cmp[row0 + k: row0 + k + m])
            eq = got == r
            nb = int((~eq).sum())
            if nb and first is None:
                f, kk, gv, wv = _first_mismatch(got, r)
                tid = (t0 + k + kk[0]) if ids is None else int(ids[k + kk[0]])
                first = f"trace {tid} policy {specs[kk[1]]}: field {f} device {gv} oracle {wv}"
            bad += nb
        if want_results:
            results.append(r)
        k += m
    tot = merge_totals(parts)
    dec = sum(t["placements"] + t["waits"] + t["rejected"] for t in tot)
    return dict(sim_s=sim_s, decisions=dec, n=count, totals=tot, mismatches=bad, first=first,
                results=np.concatenate(results) if want_results and results else None)


def run(cfg, specs, t0=0, n=0, ids=None, procs=None, cmp_path=None, want_results=False, block=4096, pool=None,
        timeout=3600):
    """Run the oracle over trace ids [t0, t0 + n) (or the int array `ids`) of config cfg on `procs` processes.

    cmp_path: a .npy file of RESULT_DTYPE rows [count, n_pol] (e.g. the device's results for the same ids, in the
    same order); every worker compares its rows element by element. Returns a dict: wall (s, the slowest worker's
    oracle time), decisions, traces, totals (per policy, merged), mismatches (count of differing (trace, policy)
    rows), first (the first mismatch, or None), procs, results (if want_results)."""
    import multiprocessing as mp

    procs = procs or (os.cpu_count() or 1)
    count = len(ids) if ids is not None else n
    procs = max(1, min(procs, count))
    bounds = [count * i // procs for i in range(procs + 1)]
    tasks = []
    for i in range(procs):
        a, b = bounds[i], bounds[i + 1]
        if ids is None:
            tasks.append((cfg, t0 + a, b - a, None, specs, block, cmp_path, a, want_results))
        else:
            tasks.append((cfg, 0, 0, np.asarray(ids[a:b], np.int64), specs, block, cmp_path, a, want_results))
    own = pool is None
    if own:
        pool = mp.get_context("spawn").Pool(procs)  # fresh interpreters (no fork after CUDA / OpenMP init)
    try:
        outs = pool.map_async(_work, tasks).get(timeout=timeout)
    finally:
        if own:
            pool.close()
            pool.join()
    first = next((o["first"] for o in outs if o["first"]), None)
    res = dict(wall=max(o["sim_s"] for o in outs), decisions=sum(o["decisions"] for o in outs), traces=count,
               totals=merge_totals([o["totals"] for o in outs]), mismatches=sum(o["mismatches"] for o in outs),
               first=first, procs=procs, per_process_decisions_per_s=float(np.mean(
                   [o["decisions"] / max(o["sim_s"], 1e-9) for o in outs])))
    if want_results:
        res["results"] = np.concatenate([o["results"] for o in outs])
    return res
