"""The seeded input generator (tracegen/): determinism, chunk independence, and the workload shapes DESIGN.md's
input recipe states. Host/device bit-equality is in test_parity_gpu.py."""
import numpy as np
import pytest

from tracegen import tracegen as tg


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_deterministic_and_chunk_independent(cfg):
    a = tg.generate_host(cfg, 50)
    b = tg.generate_host(cfg, 50)
    for x, y in zip(a, b):
        if x is not None:
            assert np.array_equal(x, y)
    # traces are a pure function of (seed, trace id): generating [20, 50) alone gives the same records
    J = tg.jobs_per_trace(cfg)
    c = tg.generate_host(cfg, 30, trace_id0=20)
    assert np.array_equal(a[0][20 * J:], c[0])


def test_config2_rodinia_shape():
    jobs, ext, off = tg.generate_host(2, 2000)
    assert ext is None and len(jobs) == 200_000 and off[-1] == 200_000
    cls = (jobs[:, 2] >> 16) & 0xFF
    assert np.all(cls == 0) and np.all((jobs[:, 2] & 0xFFFF) == 8)
    tru, est = jobs[:, 1], jobs[:, 0]
    assert tru.min() > 256 and tru.max() <= 40448
    under = np.mean(est < tru)
    assert 0.01 < under < 0.02  # 1/64 underestimates (seed OOM restarts)
    ticks = jobs[:, 3]
    assert ticks.min() >= 64 and ticks.max() < 2048


def test_config4_llm_crossing():
    # KV growth: requested + ctx crosses the 10 GB slice near iteration i_x in [24, 100]
    jobs, ext, off = tg.generate_host(4, 200)
    seed = tg.seed_of(4)
    cross = []
    for j in range(0, 800, 7):
        T = int(jobs[j, 2] & 0xFFFF)
        y, q = tg.dyn_samples(seed, j // 4, j % 4, jobs[j], ext[j], T)
        phys = y.astype(np.int64) * 65536 // q + 512
        over = np.nonzero(phys > 10240)[0]
        assert len(over) > 0
        cross.append(over[0] + 1)
    assert 15 <= np.median(cross) <= 100


def test_dyn_sample_noise_is_unbiased():
    # Irwin-Hall(4) noise: zero mean within 3 sigma/sqrt(n)
    job = np.array([10000, 65536, 4000 | (2 << 16), 10], np.uint32)
    ext = np.array([0, 0, 0, 100], np.uint32)
    y, q = tg.dyn_samples(1, 2, 3, job, ext, 4000)
    resid = y.astype(np.float64) - 10000.5  # 2 MiB rounding adds +0.5 on average
    assert abs(resid.mean()) < 3 * 100 / np.sqrt(4000)
    assert 90 < resid.std() < 110
    assert np.all(q == 65536)


def test_config_has_dynamic_table():
    # CONFIG_HAS_DYNAMIC is what lets bench.py pass MIG_TRACES_NO_DYNAMIC: it must match the generator's classes
    for cfg in [2, 3, 4, 5]:
        jobs, _, _ = tg.generate_host(cfg, 3000, trace_id0=777)
        has = bool((((jobs[:, 2] >> 16) & 0xFF) == 2).any())
        assert has == tg.CONFIG_HAS_DYNAMIC[cfg], cfg


def test_dyn_sample_noise_shape():
    # the per-iteration draw (tg_iter_bits: one 32-bit counter hash, Irwin-Hall(4) over its bytes) gives noise: symmetric, with
    # the normal's central masses (68.3% within 1 sigma, 95.4% within 2; Irwin-Hall(4): 67.8% / 95.8%), and no
    # lag-1 correlation between consecutive iterations
    sig = 1000
    job = np.array([100000, 65536, 20000 | (2 << 16), 10], np.uint32)
    ext = np.array([0, 0, 0, sig], np.uint32)
    y, _ = tg.dyn_samples(7, 11, 2, job, ext, 20000)
    r = y.astype(np.float64) - 100000.5
    s = r.std()
    assert abs(r.mean()) < 4 * sig / np.sqrt(len(r)) and 0.97 * sig < s < 1.03 * sig
    assert 0.66 < np.mean(np.abs(r) < s) < 0.70 and 0.945 < np.mean(np.abs(r) < 2 * s) < 0.965
    assert abs(np.mean(r > 0) - 0.5) < 0.02
    assert abs(np.corrcoef(r[:-1], r[1:])[0, 1]) < 0.03


def test_dyn_sample_fast_equals_reference_in_range():
    # tg_dyn_sample_fast (32-bit) == tg_dyn_sample under its bounds: b + slope*T/256 + 2^19 < 2^31, slope*T < 2^32,
    # at the edges of the noise range (sigma up to 65535) and on the configs' own dynamic jobs
    rng = np.random.default_rng(5)
    for _ in range(300):
        T = int(rng.integers(1, 4097))
        slope = int(rng.integers(0, min(2**32 // T, 2**24)))
        b = int(rng.integers(0, 2**30 - (slope * T >> 8)))
        sig = int(rng.choice([0, 1, 100, 65535, int(rng.integers(0, 65536))]))
        job = np.array([b, 65536, T | (2 << 16), 10], np.uint32)
        ext = np.array([0, 0, slope, sig | (int(rng.integers(0, 64)) << 16)], np.uint32)
        key_t, key_j = int(rng.integers(0, 2**40)), int(rng.integers(0, 50))
        a = tg.dyn_samples(9, key_t, key_j, job, ext, T)
        f = tg.dyn_samples(9, key_t, key_j, job, ext, T, fast=True)
        assert np.array_equal(a[0], f[0]) and np.array_equal(a[1], f[1])
