"""Pins for the oracle's scheduler / partition-manager event loop (Alg. 4 PAPER.md:597-617,
OOM restart PAPER.md:569, early restart PAPER.md:571/:757/:763, baseline PAPER.md:635-637).

Independent references: the hand-derived schedule of example W (tests/golden/config1_w.json), the throughput
ceilings the paper states (7x for 5 GB jobs PAPER.md:687, 2x for 20 GB jobs PAPER.md:684), closed-form energy,
the early-restart analogue of "6 vs 94" (example E), a pure-Python brute-force replay of every decision on tiny
queues (tests/bruteforce.py), and conservation invariants on generated traces.
"""
import json
import os

import numpy as np
import pytest

from bruteforce import Replay, fcr_table
from conftest import GOLDEN_DIR, geom_path
from oracle import oracle as orc
from tracegen import tracegen as tg

POLICY = {"BASELINE": 0, "STATIC": 1, "DYNAMIC": 2, "FUSION_FISSION": 3, "SCHEME_A": 4}


def spec_of(name):
    with open(geom_path(name)) as f:
        return json.load(f)


def w_fixture():
    with open(os.path.join(GOLDEN_DIR, "config1_w.json")) as f:
        fx = json.load(f)
    tr = [tg.pack_job(j["est_gb"] * 1024, j["true_gb"] * 1024, j["iters"], 0, j["iter_ticks"]) for j in fx["jobs_gb"]]
    return fx, tg.pack_traces([tr])


@pytest.mark.parametrize("pname", list(POLICY))
def test_example_w(pname):
    fx, (jobs, ext, off) = w_fixture()
    g = orc.Geometry(geom_path(fx["geometry"]))
    r, recs = orc.simulate(g, jobs, ext, off, orc.policy(kind=POLICY[pname], **fx["policy_common"]), records=True)
    r = r[0, 0]
    for k, v in fx["expected"][pname].items():
        if isinstance(v, int):
            assert int(r[k]) == v, (pname, k)
    dec = int(r["placements"]) + int(r["waits"]) + int(r["rejected"])
    assert dec == (9 if pname == "SCHEME_A" else 15)  # 15 head evaluations under Scheme B policies
    if pname == "SCHEME_A":
        assert [d["tick"] for d in recs if d["kind"] == "LAYOUT"] == [0, 80, 220]  # 3 layouts
    if pname == "FUSION_FISSION":
        got = [(d["tick"], d["job"], d["kind"], d["start"]) for d in recs if d["kind"] not in ("COMPLETE",)]
        assert got[:4] == [(0, 0, "ALLOC", 2), (0, 1, "ALLOC", 1), (0, 2, "ALLOC", 0), (0, 3, "WAIT", 15)]
        assert (160, 4, "OOM", 3) in got and (160, 7, "REUSE", 3) in got and (180, 4, "RECONF", 2) in got
    # FF vs BASELINE: throughput 450/220, energy 58500/27100


def test_throughput_ceilings():
    # 7 identical 5 GB jobs -> 7.00x; 2 identical 20 GB jobs -> 2.00x.
    g = orc.Geometry(geom_path("a100-40gb"))
    for n, gb in [(7, 4), (2, 19)]:
        tr = [tg.pack_job(gb * 1024, gb * 1024, 10, 0, 1000) for _ in range(n)]
        jobs, ext, off = tg.pack_traces([tr])
        kw = dict(ctx_mib=512, reconfig_ticks=0)
        ff = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, **kw))[0, 0]
        dyn = orc.simulate(g, jobs, ext, off, orc.policy(kind=2, **kw))[0, 0]
        sa = orc.simulate(g, jobs, ext, off, orc.policy(kind=4, **kw))[0, 0]
        base = orc.simulate(g, jobs, ext, off, orc.policy(kind=0, **kw))[0, 0]
        assert base["makespan"] / ff["makespan"] == pytest.approx(float(n), abs=0.01)
        assert base["makespan"] / dyn["makespan"] == pytest.approx(float(n), abs=0.01)
        assert base["makespan"] / sa["makespan"] == pytest.approx(float(n), abs=0.01)  # SPEC.md:481 (Scheme A)


def test_energy_closed_form():
    # single 10 s job on a flat 100 W GPU -> 1000 J; general: idle*makespan + w*sum(compute*len).
    g = orc.Geometry(geom_path("a100-40gb"))
    jobs, ext, off = tg.pack_traces([[tg.pack_job(1024, 1024, 10, 0, 1000)]])
    r = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, idle_w=100, w_per_slice=0, reconfig_ticks=0))[0, 0]
    assert r["makespan"] == 10000 and r["energy_wticks"] * 1e-3 == 1000.0
    r = orc.simulate(g, jobs, ext, off, orc.policy(kind=0, idle_w=30, w_per_slice=25, reconfig_ticks=0))[0, 0]
    assert r["energy_wticks"] == 30 * 10000 + 25 * 7 * 10000  # baseline uses all 7 compute slices


def dyn_job(b, slope, T, ticks, sigma=0, qslope=0, ws=0):
    return tg.pack_job(b, 65536, T, tg_dynamic(), ticks, ws=ws, slope_q8=slope * 256, sigma=sigma, qslope=qslope)


def tg_dynamic():
    return 2


def test_early_restart_example_E():
    # Example E: req_i = 1000 + 100 i, T = 50, 10 ticks/iter, starts on 1g.5gb (5120 MiB,
    # PAPER.md:757). Without prediction: OOM at iteration 42 (5200 > 5120) -> rerun on 2g.10gb. With prediction:
    # converged at n = 6 with 6000 > 5120 -> PREEMPT at 60 ticks. Wasted iterations 6 vs 42 ("6 vs 94").
    g = orc.Geometry(geom_path("a100-40gb"))
    jobs, ext, off = tg.pack_traces([[dyn_job(1000, 100, 50, 10)]])
    kw = dict(ctx_mib=0, reconfig_ticks=0)
    r, recs = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, **kw), records=True)
    assert [(d["tick"], d["kind"], d["profile"]) for d in recs] == [
        (0, "ALLOC", 0), (420, "OOM", 0), (420, "ALLOC", 1), (920, "COMPLETE", 1)]
    assert r[0, 0]["busy_slice_ticks"] == 420 * 1 + 500 * 2
    r, recs = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, flags=orc.EARLY_RESTART, **kw), records=True)
    assert [(d["tick"], d["kind"], d["profile"]) for d in recs] == [
        (0, "ALLOC", 0), (60, "PREEMPT", 0), (60, "ALLOC", 1), (560, "COMPLETE", 1)]
    assert r[0, 0]["preempts"] == 1 and r[0, 0]["ooms"] == 0 and r[0, 0]["makespan"] == 560


def test_head_of_line_wait():
    # "if a workload that occupies half the GPU is running and the next job requires the full GPU,
    # scheme B would wait for the first workload to finish, even though there might be workloads that can fit".
    g = orc.Geometry(geom_path("a100-40gb"))
    tr = [tg.pack_job(15000, 15000, 1, 0, 1000), tg.pack_job(35000, 35000, 1, 0, 100), tg.pack_job(1000, 1000, 1, 0, 10)]
    jobs, ext, off = tg.pack_traces([tr])
    _, recs = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, reconfig_ticks=0), records=True)
    starts = {d["job"]: d["tick"] for d in recs if d["kind"] in ("ALLOC", "RECONF", "REUSE")}
    assert starts[1] == 1000 and starts[2] == 1100  # the 5 GB job waits behind the 40 GB head (not at t=0)


def test_merge_and_split():
    g = orc.Geometry(geom_path("a100-40gb"))
    # split: an idle 7g is destroyed to create a 1g at the argmax slot
    tr = [tg.pack_job(30000, 30000, 1, 0, 100), tg.pack_job(1000, 1000, 1, 0, 100)]
    jobs, ext, off = tg.pack_traces([tr])
    _, recs = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, reconfig_ticks=0), records=True)
    assert (100, "RECONF", 6, 1) in [(d["tick"], d["kind"], d["start"], d["n_destroyed"]) for d in recs]
    # merge: two idle 1g are merged into a 2g
    tr = [tg.pack_job(1000, 1000, 1, 0, 100)] * 7 + [tg.pack_job(8000, 8000, 1, 0, 100)]
    jobs, ext, off = tg.pack_traces([tr])
    _, recs = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, reconfig_ticks=0), records=True)
    last = [d for d in recs if d["job"] == 7 and d["kind"] == "RECONF"][0]
    assert last["n_destroyed"] == 2 and last["profile"] == 1


def test_failed_and_rejected_and_empty():
    g = orc.Geometry(geom_path("a100-40gb"))
    tr = [tg.pack_job(30000, 50000, 3, 0, 10),  # fits 7g by estimate, true 50 GB: OOM on 40 GB -> FAILED
          tg.pack_job(50000, 50000, 3, 0, 10)]  # estimate above the GPU: REJECTED
    jobs, ext, off = tg.pack_traces([tr, []])
    r = orc.simulate(g, jobs, ext, off, [orc.policy(kind=k) for k in range(4)])
    for p in range(4):
        if p == 1:  # STATIC: no layout slice holds 40 GB -> both rejected (R11)
            assert r[0, p]["failed"] == 0 and r[0, p]["rejected"] == 2
        else:
            assert r[0, p]["failed"] == 1 and r[0, p]["rejected"] == 1 and r[0, p]["completed"] == 0
        e = r[1, p]
        assert e["makespan"] == 0 and e["n_jobs"] == 0 and e["decision_hash"] == 0xcbf29ce484222325


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_conservation_invariants_generated(cfg):
    n = 60
    jobs, ext, off = tg.generate_host(cfg, n)
    g = orc.Geometry(geom_path(tg.CONFIG_GEOMETRY[cfg]))
    pols = [orc.policy(kind=k) for k in range(4)] + [orc.policy(kind=3, flags=orc.EARLY_RESTART)]
    r = orc.simulate(g, jobs, ext, off, pols, seed=tg.seed_of(cfg))  # oracle asserts no overlap / capacity inside
    assert np.all(r["completed"] + r["rejected"] + r["failed"] == r["n_jobs"])
    assert np.all(r["restarts"] == r["ooms"] - r["failed"] + r["preempts"])
    assert np.all(r["energy_wticks"] == 30 * r["makespan"].astype(np.uint64) + 25 * r["busy_slice_ticks"])
    assert np.all(r["preempts"][:, :4] == 0)  # only the early-restart policy preempts
    # determinism
    r2 = orc.simulate(g, jobs, ext, off, pols, seed=tg.seed_of(cfg))
    assert np.array_equal(r, r2)


@pytest.mark.parametrize("cfg", [2, 3, 5])
def test_fifo_start_order(cfg):
    # Scheme B fairness: first starts are in queue order (head-of-line); requeues go to the tail.
    jobs, ext, off = tg.generate_host(cfg, 8)
    g = orc.Geometry(geom_path(tg.CONFIG_GEOMETRY[cfg]))
    for k in range(4):
        for t in range(8):
            _, recs = orc.simulate(g, jobs, ext, off, orc.policy(kind=k), seed=tg.seed_of(cfg), t0=t, t1=t + 1,
                                   records=True)
            first = []
            for d in recs:
                if d["kind"] in ("REUSE", "ALLOC", "RECONF", "PLACE_STATIC", "PLACE_BASELINE", "REJECT") and \
                        d["job"] not in first:
                    first.append(d["job"])
            assert first == sorted(first)


@pytest.mark.parametrize("geo,cfg", [("a30-24gb", None), ("a100-40gb", 2), ("a100-40gb", 5)])
def test_bruteforce_replay_tiny_queues(geo, cfg):
    # Every decision on tiny queues equals the brute-force optimum over all candidate successors, and only valid
    # partition states are visited (north_star: brute-force enumeration of every reachable partition state).
    spec = spec_of(geo)
    S, fcr = fcr_table(spec)
    g = orc.Geometry(spec)
    rng = np.random.default_rng(11)
    slot = spec["slot_mib"]
    traces = []
    if cfg is None:
        for _ in range(300):
            tr = []
            for _ in range(int(rng.integers(1, 5))):
                est = int(rng.integers(1, spec["total_memory_slots"] * slot))
                tru = est if rng.random() < 0.7 else int(rng.integers(1, spec["total_memory_slots"] * slot + 2000))
                tr.append(tg.pack_job(est, tru, int(rng.integers(1, 4)), 0, int(rng.integers(1, 6)) * 10))
            traces.append(tr)
        jobs, ext, off = tg.pack_traces(traces)
        seed = 0
    else:
        jobs, ext, off = tg.generate_host(cfg, 40)
        seed = tg.seed_of(cfg)
    visited = set()
    for k in range(4):
        for flags in ([0, 1] if k == 3 else [0]):
            pol = orc.policy(kind=k, flags=flags, ctx_mib=0 if cfg is None else 512, reconfig_ticks=0 if cfg is None else 500)
            for t in range(len(off) - 1):
                _, recs = orc.simulate(g, jobs, ext, off, pol, seed=seed, t0=t, t1=t + 1, records=True)
                rp = Replay(spec, k, fcr)
                for d in recs:
                    rp.step(d)
                visited |= set(rp.visited)
    assert visited <= set(S)


def test_scheme_a_reconfigurations_equal_groups():
    # on an OOM-free mix Scheme A reconfigures once per size group present
    g = orc.Geometry(geom_path("a100-40gb"))
    rng = np.random.default_rng(4)
    for _ in range(30):
        sizes = rng.choice([3000, 8000, 15000, 30000], size=int(rng.integers(1, 25)))
        tr = [tg.pack_job(int(m), int(m), 1, 0, int(rng.integers(10, 500))) for m in sizes]
        jobs, ext, off = tg.pack_traces([tr])
        r, recs = orc.simulate(g, jobs, ext, off, orc.policy(kind=4), records=True)
        groups = len({int(g.tight_fit(int(m) + 512)) if g.mem[g.tight_fit(int(m) + 512)] != 20480 else 2
                      for m in sizes})
        assert sum(d["kind"] == "LAYOUT" for d in recs) == groups
        assert r[0, 0]["ooms"] == 0 and r[0, 0]["completed"] == len(sizes)


def test_scheme_a_vs_b_directions():
    # Scheme A >= Scheme B on heterogeneous Ht1-style mixes (B waits head-of-line);
    # the Ml3 corner case (only large jobs, two 20 GB halves, static division) favours Scheme B.
    g = orc.Geometry(geom_path("a100-40gb"))
    rng = np.random.default_rng(9)
    wins = 0
    for _ in range(40):
        kinds = ["s"] * 11 + ["m"] * 2 + ["f"] * 2  # Ht1: 11 small, 2 medium, 2 full-GPU jobs
        rng.shuffle(kinds)
        mem = {"s": 3000, "m": 8000, "f": 30000}
        dur = {"s": 700, "m": 1100, "f": 2000}  # equal total time per group
        tr = [tg.pack_job(mem[k], mem[k], 1, 0, dur[k]) for k in kinds]
        jobs, ext, off = tg.pack_traces([tr])
        a, b = orc.simulate(g, jobs, ext, off, [orc.policy(kind=4), orc.policy(kind=3)])[0]
        wins += a["makespan"] <= b["makespan"]
    assert wins >= 36
    worse = 0
    for _ in range(40):  # Ml3: 18 large jobs with unequal durations
        tr = [tg.pack_job(15000, 15000, 1, 0, int(d)) for d in rng.integers(100, 2000, 18)]
        jobs, ext, off = tg.pack_traces([tr])
        a, b = orc.simulate(g, jobs, ext, off, [orc.policy(kind=4), orc.policy(kind=3)])[0]
        worse += b["makespan"] <= a["makespan"]
    assert worse >= 36


def test_wave_time_closed_form():
    # MIG_WAVE_TIME (R31 variant): A100 1g = 14 SMs x 64 warps = 896 resident warps, full = 6272.
    # A job of W = 6272 warps is one wave on the full GPU and seven on a 1g slice: its 100-tick iteration takes
    # 700 ticks there. With warp folding the tight fit keeps the wave count (7g) and the iteration stays 100.
    g = orc.Geometry(geom_path("a100-40gb"))
    jobs, ext, off = tg.pack_traces([[tg.pack_job(1000, 1000, 1, 0, 100, warps=6272)]])
    kw = dict(ctx_mib=0, reconfig_ticks=0)
    r = orc.simulate(g, jobs, ext, off, [orc.policy(kind=3, flags=orc.WAVE_TIME, **kw),
                                         orc.policy(kind=3, flags=orc.WAVE_TIME | orc.WARP_FOLD, **kw),
                                         orc.policy(kind=3, **kw), orc.policy(kind=0, flags=orc.WAVE_TIME, **kw)])[0]
    assert [int(x["makespan"]) for x in r] == [700, 100, 100, 100]
    assert int(r[0]["busy_slice_ticks"]) == 700 * 1 and int(r[1]["busy_slice_ticks"]) == 100 * 7
    # 3g (2688) vs 4g (3584): W = 3000 is 2 waves on 3g, 1 on 4g and on the full GPU
    jobs, ext, off = tg.pack_traces([[tg.pack_job(15000, 15000, 1, 0, 100, warps=3000)]])
    r = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, flags=orc.WAVE_TIME, **kw))[0, 0]
    assert int(r["makespan"]) == 200  # tight fit = 3g (fewer compute), two waves


def test_memory_utilisation_and_wasted_time():
    # PAPER.md:675 memory utilisation; one constant 4.7 GB job alone on a 40 GB GPU for the whole run
    # -> 4.7 / 40 = 0.1175 of the GPU memory
    g = orc.Geometry(geom_path("a100-40gb"))
    mib = int(4.7 * 1024)
    jobs, ext, off = tg.pack_traces([[tg.pack_job(mib, mib, 10, 0, 100)]])
    r = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, ctx_mib=0, reconfig_ticks=0))[0, 0]
    assert r["mem_mib_ticks"] / (40960 * r["makespan"]) == pytest.approx(0.1175, abs=2e-4)
    # example E: wasted run time 420 ticks (OOM at iteration 42) without prediction, 60 with early restart
    # ("avoids nearly the entire wasted execution span")
    jobs, ext, off = tg.pack_traces([[dyn_job(1000, 100, 50, 10)]])
    kw = dict(ctx_mib=0, reconfig_ticks=0)
    a = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, **kw))[0, 0]
    b = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, flags=orc.EARLY_RESTART, **kw))[0, 0]
    assert (int(a["wasted_ticks"]), int(b["wasted_ticks"])) == (420, 60)
    # memory integral of the dynamic run: sum over iterations of (1000 + 100 i) x 10 ticks
    assert int(b["mem_mib_ticks"]) == 10 * (sum(1000 + 100 * i for i in range(1, 7)) +
                                            sum(1000 + 100 * i for i in range(1, 51)))


# ---- PCIe contention (reading R39) ----

def _pcie_run(geo, jobs_list, kind, flags=orc.PCIE, reconfig=0):
    jobs, ext, off = tg.pack_traces([jobs_list])
    g = orc.Geometry(geom_path(geo))
    return orc.simulate(g, jobs, ext, off, orc.policy(kind=kind, flags=flags, ctx_mib=0, reconfig_ticks=reconfig))[0, 0]


@pytest.mark.parametrize("kind", [0, 1, 2, 3, 4])
def test_pcie_zero_fraction_changes_nothing(kind):
    """"transfer_fraction 0 for all -> no slowdown regardless of concurrency": with F = 0 the re-timed
    event loop reproduces the plain one field for field (decision hash included), on generated config-5 traces."""
    jobs, ext, off = tg.generate_host(5, 40)
    g = orc.Geometry(geom_path("a100-40gb"))
    a = orc.simulate(g, jobs, ext, off, orc.policy(kind=kind))
    b = orc.simulate(g, jobs, ext, off, orc.policy(kind=kind, flags=orc.PCIE))
    for f in orc.RESULT_DTYPE.names:
        assert np.array_equal(a[f], b[f]), f


def test_pcie_seven_transfer_jobs_closed_form():
    """7 identical 5 GB jobs with transfer fraction F/256 on the seven 1g.5gb slices run concurrently, each
    advancing at 2^24 / (256 + 6F) units of 2^-16 ticks per tick: the per-job runtime ratio is (1 - f) + 7f
    (S:381), here F = 51 (f ~ 0.2): ratio 2.2, batch throughput vs one-at-a-time 7 / 2.2 ~ 3.18 (the
    mechanism behind the paper's 1.92x instead of 7x for Needleman-Wunsch)."""
    D, F = 1000, 51
    job = tg.pack_job(4096, 4096, 10, 0, D // 10, xfer=F)
    rho = (1 << 24) // (256 - F + F * 7)
    end = -(-D * 65536 // rho)
    r = _pcie_run("a100-40gb", [job] * 7, kind=3)
    assert r["makespan"] == end == 2196
    assert r["busy_slice_ticks"] == 7 * end and r["completed"] == 7
    base = _pcie_run("a100-40gb", [job] * 7, kind=0)
    assert base["makespan"] == 7 * D  # one run at a time: c = 1, no slowdown
    assert abs(base["makespan"] / r["makespan"] - 3.19) < 0.01


def test_pcie_single_transfer_run_and_mixed_fractions():
    """c counts only transferring runs: a job with F > 0 next to F = 0 jobs runs at full speed; two F = 128 jobs
    share: 2^24 / 384 = 43690 per tick, 1000 ticks of work end at ceil(65536000 / 43690) = 1501."""
    a = tg.pack_job(4096, 4096, 10, 0, 100, xfer=128)
    b = tg.pack_job(4096, 4096, 10, 0, 300, xfer=0)
    r = _pcie_run("a100-40gb", [a, b], kind=3)
    assert r["makespan"] == 3000 and r["busy_slice_ticks"] == 1000 + 3000
    r = _pcie_run("a100-40gb", [a, a], kind=3)
    assert r["makespan"] == 1501 and r["busy_slice_ticks"] == 2 * 1501


def test_pcie_retime_when_a_transfer_run_starts_late():
    """Re-timing at a start (STATIC layout 4g@0, 2g@4, 1g@6 of A100-40GB): A (4 GB, F = 128, 1000 ticks) runs on
    1g@6 from 0; C (8 GB, F = 0) on 2g@4 and D (15 GB, F = 0) on 4g@0 run 400 ticks; B (8 GB, F = 128, 1000 ticks)
    waits and starts at 400 on 2g@4. A: 400 ticks alone, then 65536000 - 400*65536 = 39321600 units at
    2^24/384 = 43690 per tick -> ends at 400 + ceil(900.01) = 1301. B: 901 ticks shared leave
    65536000 - 901*43690 = 26171310 units, alone again at 65536 per tick -> ends at 1301 + 400 = 1701."""
    A = tg.pack_job(4096, 4096, 10, 0, 100, xfer=128)
    C = tg.pack_job(8192, 8192, 4, 0, 100)
    D = tg.pack_job(15360, 15360, 4, 0, 100)
    B = tg.pack_job(8192, 8192, 10, 0, 100, xfer=128)
    r = _pcie_run("a100-40gb", [A, C, D, B], kind=1)
    assert r["completed"] == 4 and r["makespan"] == 1701
    assert r["busy_slice_ticks"] == 1 * 1301 + 2 * 400 + 4 * 400 + 2 * (1701 - 400)
    assert r["turnaround_sum"] == 1301 + 400 + 400 + 1701
    plain = _pcie_run("a100-40gb", [A, C, D, B], kind=1, flags=0)
    assert plain["makespan"] == 1400


# ---- arrival streams (reading R40; R34's batch arrival is the paper's setting) ----

@pytest.mark.parametrize("kind", [0, 1, 2, 3])
@pytest.mark.parametrize("flags", [0, 1, 16])
def test_arrivals_at_zero_equal_batch(kind, flags):
    """Every job arriving at t = 0 is the batch setting: identical results, decision hash included."""
    jobs, ext, off = tg.generate_host(5, 30)
    g = orc.Geometry(geom_path("a100-40gb"))
    a = orc.simulate(g, jobs, ext, off, orc.policy(kind=kind, flags=flags))
    b = orc.simulate(g, jobs, ext, off, orc.policy(kind=kind, flags=flags), arrival=np.zeros(len(jobs), np.uint32))
    for f in orc.RESULT_DTYPE.names:
        assert np.array_equal(a[f], b[f]), f


def test_arrival_waits_then_fuses():
    """A (5 GB, 100 ticks) arrives at 0, B (40 GB, 50 ticks) at 10. FUSION_FISSION, ctx = reconfig = 0:
    t=0 A ALLOC 1g@6; t=10 B's arrival wakes the scheduler: B WAIT (the whole GPU overlaps busy A); t=100 A
    COMPLETE, B RECONF 7g@0 destroying A's idle slice; t=150 B COMPLETE. Turnaround 100 + 140; energy
    30*150 + 25*(1*100 + 7*50) = 15750 W*ticks."""
    A = tg.pack_job(4096, 4096, 10, 0, 10)
    B = tg.pack_job(40960, 40960, 5, 0, 10)
    jobs, ext, off = tg.pack_traces([[A, B]])
    g = orc.Geometry(geom_path("a100-40gb"))
    r, recs = orc.simulate(g, jobs, ext, off, orc.policy(kind=3, ctx_mib=0, reconfig_ticks=0), records=True,
                           arrival=np.array([0, 10], np.uint32))
    r = r[0, 0]
    got = [(x["tick"], x["job"], x["kind"], x["start"], x["n_destroyed"]) for x in recs]
    assert got == [(0, 0, "ALLOC", 6, 0), (10, 1, "WAIT", 15, 0), (100, 0, "COMPLETE", 6, 0),
                   (100, 1, "RECONF", 0, 1), (150, 1, "COMPLETE", 0, 0)]
    assert r["makespan"] == 150 and r["turnaround_sum"] == 100 + 140 and r["energy_wticks"] == 15750
    assert r["placements"] == 2 and r["waits"] == 1 and r["creates"] == 2 and r["destroys"] == 1


def test_arrival_gap_idles_the_gpu():
    """A (10 ticks) at 0, B (10 ticks) at 1000: the GPU idles in between; makespan 1010, turnaround 10 + 10,
    energy 30*1010 + 25*(10 + 10)."""
    A = tg.pack_job(4096, 4096, 1, 0, 10)
    jobs, ext, off = tg.pack_traces([[A, A]])
    g = orc.Geometry(geom_path("a100-40gb"))
    for kind in (0, 2, 3):
        r = orc.simulate(g, jobs, ext, off, orc.policy(kind=kind, ctx_mib=0, reconfig_ticks=0),
                         arrival=np.array([0, 1000], np.uint32))[0, 0]
        comp = 7 if kind == 0 else 1
        assert r["makespan"] == 1010 and r["turnaround_sum"] == 20
        assert r["energy_wticks"] == 30 * 1010 + 25 * comp * 20


def test_arrivals_spaced_beyond_durations_run_alone():
    """Arrival gaps longer than every job: each runs alone from its arrival; makespan = last arrival + its run;
    turnaround = sum of the runs (S:386 'turnaround = mean(completion - arrival)')."""
    rng = np.random.default_rng(3)
    js, arr, t = [], [], 0
    for _ in range(12):
        it, ticks = int(rng.integers(1, 6)), int(rng.integers(1, 100))
        js.append(tg.pack_job(4096, 4096, it, 0, ticks))
        arr.append(t)
        last = it * ticks
        t += 600
    jobs, ext, off = tg.pack_traces([js])
    g = orc.Geometry(geom_path("a100-40gb"))
    durs = [int(j[0][2] & 0xFFFF) * int(j[0][3]) for j in js]
    for kind in (0, 1, 2, 3):
        r = orc.simulate(g, jobs, ext, off, orc.policy(kind=kind, ctx_mib=0, reconfig_ticks=0),
                         arrival=np.array(arr, np.uint32))[0, 0]
        assert r["makespan"] == arr[-1] + durs[-1] and r["turnaround_sum"] == sum(durs) and r["waits"] == 0


def test_arrival_rejected_after_last_completion_extends_makespan():
    """R40: makespan is the last tick with an end or an arrival. A job no slice can hold, arriving after the last
    completion, is rejected at its arrival tick, which ends the run: A (10 ticks) at 0, B (50 GB, too large for
    A100-40GB) at 500 -> makespan 500, one REJECT at 500."""
    A = tg.pack_job(4096, 4096, 1, 0, 10)
    B = tg.pack_job(51200, 51200, 1, 0, 10)
    jobs, ext, off = tg.pack_traces([[A, B]])
    g = orc.Geometry(geom_path("a100-40gb"))
    for kind in (0, 1, 2, 3):
        r, recs = orc.simulate(g, jobs, ext, off, orc.policy(kind=kind, ctx_mib=0, reconfig_ticks=0), records=True,
                               arrival=np.array([0, 500], np.uint32))
        assert r[0, 0]["makespan"] == 500 and r[0, 0]["rejected"] == 1 and r[0, 0]["completed"] == 1
        assert recs[-1]["tick"] == 500 and recs[-1]["kind"] == "REJECT"
