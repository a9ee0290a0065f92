"""GPU parity: the CUDA path (libmig.so through its C ABI) against the CPU oracle, element by element.

Bar (north_star): every integer field of every (trace, policy) result — makespan, counts, energy W*ticks,
turnaround, busy slice-ticks and the 64-bit hash of every placement decision and event time — is bit-exact.
Estimate doubles (phi, a, sigma) must agree within 1e-6 relative (they are expected to be bit-identical: both
sides run the same canonical IEEE sequence).
"""
import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN_DIR, geom_path
from oracle import oracle as orc
from tracegen import tracegen as tg

import paper_2508_18556_b200 as mig

pytestmark = pytest.mark.gpu

SPECS = [dict(kind=0), dict(kind=1), dict(kind=2), dict(kind=3), dict(kind=3, flags=1), dict(kind=4),
         dict(kind=4, flags=1)]
ESTIMATE_FIELDS = ["req0_mib", "pred_mib", "conv_iter", "n_levels", "fe", "phi", "a", "sigma", "mem_fe",
                   "mem_conv", "mem_T"]


def run_pair(geo, jobs, ext, off, specs, seed=0, common=None, max_jobs=None, arrival=None):
    common = common or {}
    g = mig.mig_geometry_load(f"builtin:{geo}")
    og = orc.Geometry(geom_path(geo))
    pols = [mig.policy(g, **s, **common) for s in specs]
    opols = [orc.policy(**s, **common) for s in specs]
    tr = mig.traces_from_numpy(jobs, ext, off, seed=seed, max_jobs=max_jobs, arrival=arrival)
    res, tot = mig.mig_simulate(g, tr, pols)
    torch.cuda.synchronize()
    got = mig.results_numpy(res, len(pols))
    want = orc.simulate(og, jobs, ext, off, opols, seed=seed, arrival=arrival)
    return got, want, mig.totals_numpy(tot)


def random_arrivals(rng, off, spread):
    """Non-decreasing arrival ticks per trace (R40): sorted uniform draws in [0, spread), some traces all at 0."""
    arr = np.zeros(int(off[-1]), np.uint32)
    for t in range(len(off) - 1):
        a, b = int(off[t]), int(off[t + 1])
        if b > a and rng.random() < 0.8:
            arr[a:b] = np.sort(rng.integers(0, spread, b - a))
    return arr


def assert_same(got, want):
    assert got.shape == want.shape
    for f in orc.RESULT_DTYPE.names:
        if not np.array_equal(got[f], want[f]):
            bad = tuple(np.argwhere(got[f] != want[f])[0])
            pytest.fail(f"field {f} differs at (trace, policy) {bad}: gpu {got[f][bad]} oracle {want[f][bad]}")


def check_totals(got, tot):
    for p in range(got.shape[1]):
        r = got[:, p]
        t = tot[p]
        assert t["n_traces"] == len(r) and t["error_flags"] == 0
        for f in ["n_jobs", "completed", "rejected", "failed", "ooms", "preempts", "restarts", "placements",
                  "waits", "creates", "destroys", "energy_wticks", "turnaround_sum", "busy_slice_ticks",
                  "mem_mib_ticks", "wasted_ticks"]:
            assert int(t[f]) == int(r[f].astype(np.uint64).sum()), f
        assert int(t["makespan_sum"]) == int(r["makespan"].astype(np.uint64).sum())
        assert int(t["makespan_max"]) == int(r["makespan"].max(initial=0))
        assert int(t["decision_hash_sum"]) == int(r["decision_hash"].astype(np.uint64).sum(dtype=np.uint64))


def test_config1_example_w_all_policies():
    with open(os.path.join(GOLDEN_DIR, "config1_w.json")) as f:
        fx = json.load(f)
    tr = [tg.pack_job(j["est_gb"] * 1024, j["true_gb"] * 1024, j["iters"], 0, j["iter_ticks"]) for j in fx["jobs_gb"]]
    jobs, ext, off = tg.pack_traces([tr])
    specs = [dict(kind=k) for k in range(5)]
    got, want, tot = run_pair("a30-24gb", jobs, ext, off, specs, common=fx["policy_common"])
    assert got[0, 4]["makespan"] == 270 and got[0, 4]["energy_wticks"] == 28600  # Scheme A
    assert_same(got, want)
    assert got[0, 3]["makespan"] == 220 and got[0, 3]["energy_wticks"] == 27100
    check_totals(got, tot)


@pytest.mark.parametrize("cfg,n", [(2, 400), (3, 600), (4, 3000), (5, 300)])
def test_generated_configs_all_policies(cfg, n):
    jobs, ext, off = tg.generate_host(cfg, n)
    got, want, tot = run_pair(tg.CONFIG_GEOMETRY[cfg], jobs, ext, off, SPECS, seed=tg.seed_of(cfg))
    assert_same(got, want)
    check_totals(got, tot)


@pytest.mark.parametrize("cfg,n", [(3, 300), (4, 2000), (5, 200)])
def test_estimates_match_oracle(cfg, n):
    jobs, ext, off = tg.generate_host(cfg, n)
    geo = tg.CONFIG_GEOMETRY[cfg]
    g = mig.mig_geometry_load(f"builtin:{geo}")
    og = orc.Geometry(geom_path(geo))
    tr = mig.traces_from_numpy(jobs, ext, off, seed=tg.seed_of(cfg))
    est = mig.estimates_numpy(mig.mig_estimate_memory(g, tr, mig.policy(g)))
    want = orc.estimate(og, jobs, ext, off, orc.policy(), seed=tg.seed_of(cfg))
    for f in ["req0_mib", "pred_mib", "conv_iter", "n_levels", "fe", "mem_fe", "mem_conv", "mem_T"]:
        assert np.array_equal(est[f], want[f]), f
    for f in ["phi", "a", "sigma"]:
        np.testing.assert_allclose(est[f], want[f], rtol=1e-6, atol=1e-9)
        assert np.array_equal(est[f], want[f]), f"{f} not bit-identical"
    dyn = ((jobs[:, 2] >> 16) & 0xFF) == 2
    assert dyn.any() and (est["conv_iter"][dyn] > 0).any()


def random_tiny_traces(rng, geo_spec, n_traces, max_len, dyn_frac=0.3, xfer=False):
    slot = geo_spec["slot_mib"]
    full = geo_spec["total_memory_slots"] * slot
    traces = []
    for _ in range(n_traces):
        tr = []
        for _ in range(int(rng.integers(0, max_len + 1))):
            if rng.random() < dyn_frac:
                b = int(rng.integers(100, full // 3))
                T = int(rng.integers(1, 300))
                tr.append(tg.pack_job(b, 65536, T, 2, int(rng.integers(1, 50)), ws=int(rng.integers(0, 64)),
                                      slope_q8=int(rng.integers(0, 200 * 256)), sigma=int(rng.integers(0, 200)),
                                      qslope=int(rng.integers(0, 100)),
                                      xfer=int(rng.integers(0, 256)) if xfer and rng.random() < 0.6 else 0))
            else:
                est = int(rng.integers(1, full + 4000))
                tru = est if rng.random() < 0.6 else int(rng.integers(1, full + 4000))
                tr.append(tg.pack_job(est, tru, int(rng.integers(0, 6)), int(rng.integers(0, 2)),
                                      int(rng.integers(1, 2000)), ws=int(rng.integers(0, 100)),
                                      warps=int(rng.integers(0, 20000)),
                                      xfer=int(rng.integers(0, 256)) if xfer and rng.random() < 0.6 else 0))
        traces.append(tr)
    return tg.pack_traces(traces)


@pytest.mark.parametrize("geo", ["a30-24gb", "a100-40gb", "a100-40gb-1g10", "h100-80gb", "b200-180gb"])
def test_random_ragged_traces_edge_cases(geo):
    # empty traces, ragged lengths, zero-iteration jobs, rejections, failures at the full GPU, warp folding
    spec = json.load(open(geom_path(geo)))
    rng = np.random.default_rng(5)
    jobs, ext, off = random_tiny_traces(rng, spec, 500, 40)
    specs = SPECS + [dict(kind=3, flags=3)]
    for common in [dict(ctx_mib=0, reconfig_ticks=0), dict(ctx_mib=512, reconfig_ticks=500, z=1.0)]:
        got, want, tot = run_pair(geo, jobs, ext, off, specs, seed=99, common=common)
        assert_same(got, want)
        check_totals(got, tot)


def test_max_length_trace():
    rng = np.random.default_rng(8)
    tr = []
    for _ in range(mig.MIG_MAX_JOBS_PER_TRACE):
        tr.append(tg.pack_job(int(rng.integers(1, 30000)), int(rng.integers(1, 30000)), 1, 0,
                              int(rng.integers(1, 100))))
    jobs, ext, off = tg.pack_traces([tr, [], tr[:17]])
    got, want, tot = run_pair("a100-40gb", jobs, ext, off, SPECS, max_jobs=mig.MIG_MAX_JOBS_PER_TRACE)
    assert_same(got, want)


def test_trace_longer_than_max_jobs_is_flagged():
    tr = [tg.pack_job(1000, 1000, 1, 0, 10)] * 10
    jobs, ext, off = tg.pack_traces([tr])
    g = mig.mig_geometry_load("builtin:a100-40gb")
    t = mig.traces_from_numpy(jobs, ext, off, max_jobs=4)
    _, tot = mig.mig_simulate(g, t, [mig.policy(g)])
    assert mig.totals_numpy(tot)[0]["error_flags"] & 1


def test_host_pipeline_matches_device(monkeypatch):
    monkeypatch.setenv("MIG_HOST_CHUNK_JOBS", "5000")  # force many pipelined chunks
    cfg, n = 3, 700
    jobs, ext, off = tg.generate_host(cfg, n)
    g = mig.mig_geometry_load(f"builtin:{tg.CONFIG_GEOMETRY[cfg]}")
    pols = [mig.policy(g, **s) for s in SPECS]
    hres, htot = mig.mig_simulate_host(g, jobs, ext, off, pols, seed=tg.seed_of(cfg))
    tr = mig.traces_from_numpy(jobs, ext, off, seed=tg.seed_of(cfg))
    res, tot = mig.mig_simulate(g, tr, pols)
    assert np.array_equal(hres, mig.results_numpy(res, len(pols)))
    assert np.array_equal(htot, mig.totals_numpy(tot))
    none, htot2 = mig.mig_simulate_host(g, jobs, ext, off, pols, seed=tg.seed_of(cfg), results=False)
    assert none is None and np.array_equal(htot2, htot)  # totals only (out = NULL): the same metrics


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_device_generator_equals_host(cfg):
    n = 3000
    hj, he, ho = tg.generate_host(cfg, n, trace_id0=12345)
    dj, de, do = tg.generate_device(cfg, n, trace_id0=12345)
    torch.cuda.synchronize()
    assert np.array_equal(dj.cpu().numpy().view(np.uint32), hj)
    if he is not None:
        assert np.array_equal(de.cpu().numpy().view(np.uint32), he)
    assert np.array_equal(do.cpu().numpy().view(np.uint64), ho)


@pytest.mark.parametrize("cfg,n_full,n_sample", [(2, 1_000_000, 1500), (3, 1_000_000, 1500), (4, 2_000_000, 4000),
                                               (5, 4_000_000, 800)])
def test_full_size_sampled_parity(cfg, n_full, n_sample):
    """BASELINE.json sizes (C4 at 1/5, C5 at 1/3 of its 8-GPU shard, to bound memory) in the launch configuration
    bench.py uses: device-generated traces, all policies in one call; sampled traces are regenerated on the host and
    run through the oracle."""
    geo = tg.CONFIG_GEOMETRY[cfg]
    g = mig.mig_geometry_load(f"builtin:{geo}")
    og = orc.Geometry(geom_path(geo))
    seed = tg.seed_of(cfg)
    dj, de, do = tg.generate_device(cfg, n_full)
    tr = mig.Traces(dj, de, do, n_full, seed=seed, max_jobs=tg.jobs_per_trace(cfg))
    pols = [mig.policy(g, **s) for s in SPECS]
    res, tot = mig.mig_simulate(g, tr, pols)
    torch.cuda.synchronize()
    rng = np.random.default_rng(cfg)
    idx = np.unique(np.concatenate([rng.integers(0, n_full, n_sample), [0, n_full - 1]]))
    got_all = res.view(-1, len(pols), 96)
    got = got_all[torch.from_numpy(idx).to(res.device)].cpu().numpy().view(mig.RESULT_DTYPE).reshape(-1, len(pols))
    want = np.zeros((len(idx), len(pols)), orc.RESULT_DTYPE)
    for k, t in enumerate(idx):
        hj, he, ho = tg.generate_host(cfg, 1, trace_id0=int(t))
        want[k] = orc.simulate(og, hj, he, ho, [orc.policy(**s) for s in SPECS], seed=seed, trace_id0=int(t))[0]
    assert_same(got, want)
    # totals over the whole launch equal the sum of the per-trace results
    allres = mig.results_numpy(res, len(pols))
    check_totals(allres, mig.totals_numpy(tot))


@pytest.mark.parametrize("cfg,n", [(3, 300), (5, 200)])
def test_ewma_variant_parity(cfg, n):
    # MIG_EWMA_REUSE (R36, north_star only; parity unpinned by the paper): device == oracle bit for bit
    jobs, ext, off = tg.generate_host(cfg, n)
    specs = [dict(kind=3, flags=1 | 4), dict(kind=2, flags=1 | 4), dict(kind=0, flags=4)]
    got, want, tot = run_pair(tg.CONFIG_GEOMETRY[cfg], jobs, ext, off, specs, seed=tg.seed_of(cfg))
    assert_same(got, want)
    geo = tg.CONFIG_GEOMETRY[cfg]
    g = mig.mig_geometry_load(f"builtin:{geo}")
    og = orc.Geometry(geom_path(geo))
    tr = mig.traces_from_numpy(jobs, ext, off, seed=tg.seed_of(cfg))
    est = mig.estimates_numpy(mig.mig_estimate_memory(g, tr, mig.policy(g, flags=4)))
    ref = orc.estimate(og, jobs, ext, off, orc.policy(flags=4), seed=tg.seed_of(cfg))
    for f in ESTIMATE_FIELDS:
        assert np.array_equal(est[f], ref[f]), f


@pytest.mark.parametrize("geo", ["a100-40gb", "a30-24gb"])
def test_wave_time_and_fold_variants(geo):
    # MIG_WAVE_TIME (R31 variant) x MIG_WARP_FOLD x early restart, all policy kinds, random ragged traces with warps
    spec = json.load(open(geom_path(geo)))
    jobs, ext, off = random_tiny_traces(np.random.default_rng(21), spec, 400, 30)
    specs = [dict(kind=0, flags=8), dict(kind=1, flags=8), dict(kind=2, flags=8 | 2), dict(kind=3, flags=8),
             dict(kind=3, flags=8 | 2 | 1), dict(kind=4, flags=8), dict(kind=4, flags=8 | 2 | 1), dict(kind=1, flags=3)]
    got, want, tot = run_pair(geo, jobs, ext, off, specs, seed=5, common=dict(ctx_mib=128, reconfig_ticks=20))
    assert_same(got, want)
    check_totals(got, tot)


@pytest.mark.parametrize("cfg,n", [(3, 300), (4, 1000)])
def test_recorded_samples_parity(cfg, n, monkeypatch):
    # the predictor on recorded traces: explicit per-iteration samples through the C ABI
    jobs, ext, off = tg.generate_host(cfg, n)
    seed = tg.seed_of(cfg)
    smp, soff = tg.explicit_samples(jobs, ext, off, seed)
    geo = tg.CONFIG_GEOMETRY[cfg]
    g = mig.mig_geometry_load(f"builtin:{geo}")
    og = orc.Geometry(geom_path(geo))
    wrong_seed = seed ^ 0xABCDEF  # recorded samples must be what is used, not the generator
    tr = mig.traces_from_numpy(jobs, ext, off, seed=wrong_seed, samples=smp, sample_off=soff)
    est = mig.estimates_numpy(mig.mig_estimate_memory(g, tr, mig.policy(g)))
    ref = orc.estimate(og, jobs, ext, off, orc.policy(), seed=seed)  # generator with the right seed
    for f in ESTIMATE_FIELDS:
        assert np.array_equal(est[f], ref[f]), f
    pols = [mig.policy(g, **s) for s in SPECS]
    res, _ = mig.mig_simulate(g, tr, pols)
    want = orc.simulate(og, jobs, ext, off, [orc.policy(**s) for s in SPECS], seed=wrong_seed, samples=smp,
                        sample_off=soff)
    assert_same(mig.results_numpy(res, len(pols)), want)
    monkeypatch.setenv("MIG_HOST_CHUNK_JOBS", "3000")
    hres, _ = mig.mig_simulate_host(g, jobs, ext, off, pols, seed=wrong_seed, samples=smp, sample_off=soff)
    assert_same(hres, want)


@pytest.mark.parametrize("geo", ["a30-24gb", "a100-40gb", "b200-180gb"])
def test_pcie_contention_parity(geo):
    """MIG_PCIE_CONTENTION (R39): re-timed runs, start events, actual-duration power / memory / waste, on random
    ragged traces with random transfer fractions, every policy (Scheme A and early restart included), with and
    without creation delays."""
    spec = json.load(open(geom_path(geo)))
    rng = np.random.default_rng(17)
    jobs, ext, off = random_tiny_traces(rng, spec, 600, 30, xfer=True)
    specs = [dict(kind=k, flags=16) for k in range(5)] + [dict(kind=3, flags=17), dict(kind=4, flags=17),
                                                          dict(kind=2, flags=16 | 8)]
    for common in [dict(ctx_mib=0, reconfig_ticks=0), dict(ctx_mib=512, reconfig_ticks=500)]:
        got, want, tot = run_pair(geo, jobs, ext, off, specs, seed=23, common=common)
        assert_same(got, want)
        check_totals(got, tot)


def test_pcie_contention_generated_config5():
    """Config-5 traces (five policies) with transfer fractions added to the records, against the oracle."""
    jobs, ext, off = tg.generate_host(5, 300)
    rng = np.random.default_rng(29)
    jobs = jobs.copy()
    jobs[:, 2] |= (rng.integers(0, 128, len(jobs)).astype(np.uint32) << 24)
    specs = [dict(kind=k, flags=16) for k in range(5)] + [dict(kind=3, flags=17)]
    got, want, tot = run_pair(tg.CONFIG_GEOMETRY[5], jobs, ext, off, specs, seed=tg.seed_of(5))
    assert_same(got, want)
    check_totals(got, tot)
    plain = orc.simulate(orc.Geometry(geom_path(tg.CONFIG_GEOMETRY[5])), jobs, ext, off,
                         [orc.policy(**{**sp, "flags": sp["flags"] & ~16}) for sp in specs], seed=tg.seed_of(5))
    assert (plain["makespan"][:, 3] < want["makespan"][:, 3]).mean() > 0.5  # contention slows FF down
    assert np.array_equal(plain["makespan"][:, 0], want["makespan"][:, 0])  # one run at a time: never contended


@pytest.mark.parametrize("geo", ["a30-24gb", "a100-40gb", "h100-80gb"])
def test_arrival_streams_parity(geo):
    """Arrival streams (R40): random non-decreasing arrival ticks on random ragged traces, every Scheme B policy
    and BASELINE, with and without PCIe contention and creation delays; per-trace results and totals."""
    spec = json.load(open(geom_path(geo)))
    rng = np.random.default_rng(31)
    jobs, ext, off = random_tiny_traces(rng, spec, 600, 30, xfer=True)
    arrival = random_arrivals(rng, off, 3000)
    specs = [dict(kind=k) for k in range(4)] + [dict(kind=3, flags=1), dict(kind=2, flags=16),
                                                dict(kind=3, flags=17), dict(kind=0, flags=16)]
    for common in [dict(ctx_mib=0, reconfig_ticks=0), dict(ctx_mib=512, reconfig_ticks=500)]:
        got, want, tot = run_pair(geo, jobs, ext, off, specs, seed=37, common=common, arrival=arrival)
        assert_same(got, want)
        check_totals(got, tot)


def test_arrival_streams_host_pipeline_and_config2(monkeypatch):
    """Config-2 traces with arrival streams through mig_simulate_host (chunked H2D of the arrival ticks) equal the
    device call and the oracle."""
    monkeypatch.setenv("MIG_HOST_CHUNK_JOBS", "20000")
    jobs, ext, off = tg.generate_host(2, 400)
    arrival = random_arrivals(np.random.default_rng(41), off, 200000)
    specs = [dict(kind=3), dict(kind=0)]
    got, want, tot = run_pair("a100-40gb", jobs, ext, off, specs, seed=tg.seed_of(2), arrival=arrival)
    assert_same(got, want)
    g = mig.mig_geometry_load("builtin:a100-40gb")
    pols = [mig.policy(g, **sp) for sp in specs]
    hres, htot = mig.mig_simulate_host(g, jobs, ext, off, pols, seed=tg.seed_of(2), arrival=arrival)
    assert_same(hres, want)


def test_nine_profile_geometry_uses_the_group_kernel(tmp_path):
    """A geometry with more than 8 profiles (the lane kernel packs per-profile idle masks in 64 bits) runs on the
    group kernel: same parity bar, random ragged traces, Scheme B policies."""
    prof = []
    for name, c, ln, st in [("1g.a", 1, 1, list(range(7))), ("1g.b", 1, 2, [0, 2, 4, 6]), ("2g.b", 2, 2, [0, 2, 4]),
                            ("1g.c", 1, 4, [0, 4]), ("2g.c", 2, 4, [0, 4]), ("3g.c", 3, 4, [0, 4]),
                            ("4g.c", 4, 4, [0]), ("5g.d", 5, 8, [0]), ("7g.d", 7, 8, [0])]:
        prof.append({"name": name, "compute_slices": c, "memory_slots": ln, "starts": st})
    spec = {"gpu_name": "NINE", "total_memory_slots": 8, "slot_mib": 5120, "total_compute_slices": 7,
            "sms_per_slice": 14, "warps_per_sm": 64, "idle_w": 30, "w_per_slice": 25, "profiles": prof}
    path = tmp_path / "nine.json"
    path.write_text(json.dumps(spec))
    g = mig.mig_geometry_load(str(path))
    assert g.info.n_profiles == 9
    og = orc.Geometry(str(path))
    rng = np.random.default_rng(43)
    jobs, ext, off = random_tiny_traces(rng, spec, 300, 25)
    specs = [dict(kind=0), dict(kind=2), dict(kind=3), dict(kind=3, flags=1)]
    pols = [mig.policy(g, **s, ctx_mib=256, reconfig_ticks=100) for s in specs]
    tr = mig.traces_from_numpy(jobs, ext, off, seed=5)
    res, tot = mig.mig_simulate(g, tr, pols)
    torch.cuda.synchronize()
    got = mig.results_numpy(res, len(pols))
    want = orc.simulate(og, jobs, ext, off, [orc.policy(**s, ctx_mib=256, reconfig_ticks=100) for s in specs], seed=5)
    assert_same(got, want)
    check_totals(got, mig.totals_numpy(tot))


def test_cuda_graph_capture_and_replay():
    """mig_simulate is stream-ordered (scratch by cudaMallocAsync, policy launches forked onto a side stream and
    joined by events), so a call can be captured into a CUDA graph and replayed: the replays reproduce the eager
    results bit for bit, and the oracle's."""
    cfg, n = 3, 400
    jobs, ext, off = tg.generate_host(cfg, n)
    geo = tg.CONFIG_GEOMETRY[cfg]
    g = mig.mig_geometry_load(f"builtin:{geo}")
    pols = [mig.policy(g, **s) for s in SPECS]
    tr = mig.traces_from_numpy(jobs, ext, off, seed=tg.seed_of(cfg))
    res, tot = mig.mig_simulate(g, tr, pols)  # eager (also uploads the geometry tables)
    torch.cuda.synchronize()
    eager = mig.results_numpy(res, len(pols)).copy()
    out = torch.zeros_like(res)
    totals = torch.zeros_like(tot)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        mig.mig_simulate(g, tr, pols, out=out, totals=totals)
    for _ in range(3):
        out.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(mig.results_numpy(out, len(pols)), eager)
        assert torch.equal(totals, tot)
    want = orc.simulate(orc.Geometry(geom_path(geo)), jobs, ext, off, [orc.policy(**s) for s in SPECS],
                        seed=tg.seed_of(cfg))
    assert_same(eager, want)


def test_exact_division_hook():
    """k_estimate's fast physical-memory division (float estimate + one integer correction) equals integer
    division floor(y * 2^16 / q) on its whole domain's edges and on 2^24 random pairs (y < 2^18, 2^16 <= q < 2^26)."""
    rng = np.random.default_rng(7094)
    n = 1 << 24
    y = rng.integers(0, 1 << 18, n, dtype=np.uint64)
    q = rng.integers(1 << 16, 1 << 26, n, dtype=np.uint64)
    # edges: extreme y and q, exact multiples, quotients just below / above integers
    ey = np.array([0, 1, (1 << 18) - 1, (1 << 18) - 1, (1 << 18) - 1, 65535, 65536, 3, 12345], np.uint64)
    eq = np.array([1 << 16, 1 << 16, 1 << 16, (1 << 26) - 1, (1 << 16) + 1, 65536, 65537, 196608, 99999], np.uint64)
    k = rng.integers(1, 1 << 12, 1 << 20, dtype=np.uint64)
    yk = rng.integers(1, 1 << 18, k.size, dtype=np.uint64)
    qk = np.clip((yk << np.uint64(16)) // k, 1 << 16, (1 << 26) - 1).astype(np.uint64)
    ys = np.concatenate([y, ey, yk, yk, yk])
    qs = np.concatenate([q, eq, qk, np.minimum(qk + np.uint64(1), (1 << 26) - 1),
                         np.maximum(qk - np.uint64(1), 1 << 16)])
    want = (ys << np.uint64(16)) // qs
    dev = torch.device("cuda", 0)
    ty = torch.from_numpy(ys.astype(np.uint32).view(np.int32)).to(dev)
    tq = torch.from_numpy(qs.astype(np.uint32).view(np.int32)).to(dev)
    got = mig.mig_debug_phys_div(ty, tq).cpu().numpy().view(np.uint32).astype(np.uint64)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (ys[bad[:5]], qs[bad[:5]], got[bad[:5]], want[bad[:5]])


def test_no_dynamic_flag_skips_estimator_same_results():
    # MIG_TRACES_NO_DYNAMIC (include/mig.h): on static-only traces the estimator pass is skipped (one launch fewer)
    # and every result is unchanged; a DYNAMIC record under the flag is reported as MIG_ERR_BAD_RECORD
    cfg, n = 2, 3000
    jobs, ext, off = tg.generate_host(cfg, n)
    g = mig.mig_geometry_load(f"builtin:{tg.CONFIG_GEOMETRY[cfg]}")
    pols = [mig.policy(g, **s) for s in SPECS]
    tr = mig.traces_from_numpy(jobs, ext, off, seed=tg.seed_of(cfg))
    res_a, tot_a = mig.mig_simulate(g, tr, pols)
    la = mig.mig_last_launch_count()
    tr.desc.flags = mig.MIG_TRACES_NO_DYNAMIC
    res_b, tot_b = mig.mig_simulate(g, tr, pols)
    lb = mig.mig_last_launch_count()
    torch.cuda.synchronize()
    assert lb == la - 1
    assert torch.equal(res_a, res_b) and torch.equal(tot_a, tot_b)
    # a DYNAMIC job under the flag: flagged in every policy's totals
    j3, e3, o3 = tg.generate_host(3, 50)
    tr3 = mig.traces_from_numpy(j3, e3, o3, seed=tg.seed_of(3))
    tr3.desc.flags = mig.MIG_TRACES_NO_DYNAMIC
    g3 = mig.mig_geometry_load("builtin:a100-80gb")
    _, tot3 = mig.mig_simulate(g3, tr3, [mig.policy(g3, **s) for s in SPECS])
    t3 = mig.totals_numpy(tot3)
    assert ((t3["error_flags"] & 2) != 0).all()


def test_tick_overflow_flagged():
    # ticks are u32 (include/mig.h): a run whose end does not fit is flagged MIG_ERR_TICK_OVERFLOW in every policy's
    # totals (lane kernels: generic, FUSION_FISSION fast case, BASELINE fold); an in-range trace is not
    big = [tg.pack_job(1000, 1000, 4, 0, 1 << 31)]
    ok = [tg.pack_job(1000, 1000, 4, 0, 1000)]
    g = mig.mig_geometry_load("builtin:a100-40gb")
    for jobs_list, want in [(big, 4), (ok, 0)]:
        jobs, ext, off = tg.pack_traces([jobs_list])
        tr = mig.traces_from_numpy(jobs, None, off)
        _, tot = mig.mig_simulate(g, tr, [mig.policy(g, **s) for s in SPECS])
        flags = mig.totals_numpy(tot)["error_flags"]
        assert ((flags & 4) == want).all(), flags


def test_threads_and_scratch_release():
    # calls from two host threads on their own streams (each thread has its own library side stream) give the
    # single-threaded results; mig_release_scratch trims the library's private pool afterwards
    import threading

    cfg, n = 2, 2000
    jobs, ext, off = tg.generate_host(cfg, n)
    g = mig.mig_geometry_load("builtin:a100-40gb")
    pols = [mig.policy(g, **s) for s in SPECS]
    tr = mig.traces_from_numpy(jobs, ext, off, seed=tg.seed_of(cfg))
    ref, rtot = mig.mig_simulate(g, tr, pols)
    torch.cuda.synchronize()
    outs = [None, None]

    def work(k):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                outs[k] = mig.mig_simulate(g, tr, pols, stream=s)
        s.synchronize()

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for res, tot in outs:
        assert torch.equal(res, ref) and torch.equal(tot, rtot)
    mig.mig_release_scratch()


def test_recorded_trace_files(tmp_path):
    # the predictor and scheduler on recorded traces read from CSV trace files (SPEC.md S:260 format, loaded by
    # mig_samples_load_csv): every DYNAMIC job's series written as bytes and reuse ratios, read back, assembled into
    # mig_traces.samples, and simulated; identical to the oracle on the same recorded samples
    cfg, n = 3, 120
    jobs, ext, off = tg.generate_host(cfg, n)
    seed = tg.seed_of(cfg)
    smp, soff = tg.explicit_samples(jobs, ext, off, seed)
    series = []
    for j in range(len(jobs)):
        a, b = int(soff[j]), int(soff[j + 1])
        if b == a:
            series.append(None)
            continue
        p = tmp_path / f"job{j}.csv"
        rows = ["iteration,requested_bytes,reuse_ratio"]
        rows += [f"{i + 1},{int(y) * 1048576},{65536.0 / int(q)!r}" for i, (y, q) in enumerate(smp[a:b])]
        p.write_text("\n".join(rows) + "\n")
        series.append(mig.mig_samples_load_csv(str(p)))
    smp2, soff2 = mig.samples_from_series(jobs, series)
    assert np.array_equal(soff2, soff) and np.array_equal(smp2, smp[: len(smp2)])
    geo = tg.CONFIG_GEOMETRY[cfg]
    g = mig.mig_geometry_load(f"builtin:{geo}")
    og = orc.Geometry(geom_path(geo))
    tr = mig.traces_from_numpy(jobs, ext, off, seed=1, samples=smp2, sample_off=soff2)
    pols = [mig.policy(g, **s) for s in SPECS]
    res, _ = mig.mig_simulate(g, tr, pols)
    want = orc.simulate(og, jobs, ext, off, [orc.policy(**s) for s in SPECS], seed=1, samples=smp2, sample_off=soff2)
    assert_same(mig.results_numpy(res, len(pols)), want)


@pytest.mark.parametrize("geo", ["a30-24gb", "a100-40gb", "a100-40gb-1g10", "h100-80gb", "b200-180gb"])
def test_fast_kernels_random_traces_without_ext(geo):
    # traces without extension records take k_ff_lane (FUSION_FISSION), k_base_lane (BASELINE) and, for Scheme A,
    # k_sa_group: empty traces, ragged lengths, zero-iteration jobs, rejections, failures on the whole GPU, DYNAMIC
    # jobs (estimates read in the run start), every geometry (start-slot scans of 4, 7 and 8 slots)
    spec = json.load(open(geom_path(geo)))
    rng = np.random.default_rng(41)
    jobs, _, off = random_tiny_traces(rng, spec, 600, 40, dyn_frac=0.2)
    for common in [dict(ctx_mib=0, reconfig_ticks=0), dict(ctx_mib=512, reconfig_ticks=500)]:
        got, want, tot = run_pair(geo, jobs, None, off, SPECS, seed=31, common=common)
        assert_same(got, want)
        check_totals(got, tot)
    rng = np.random.default_rng(9)  # a maximum-length trace, an empty one and a short one
    tr = [tg.pack_job(int(rng.integers(1, spec["slot_mib"] * 3)), int(rng.integers(1, spec["slot_mib"] * 3)), 1, 0,
                      int(rng.integers(1, 100))) for _ in range(mig.MIG_MAX_JOBS_PER_TRACE)]
    jobs, _, off = tg.pack_traces([tr, [], tr[:17]])
    got, want, tot = run_pair(geo, jobs, None, off, SPECS, max_jobs=mig.MIG_MAX_JOBS_PER_TRACE)
    assert_same(got, want)
