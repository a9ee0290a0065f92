"""Arithmetic claims the CUDA path relies on (DESIGN.md §6 k_estimate), checked on the CPU at the domain's edges and
on random samples.

k_estimate maps a requested MiB y (< 2^18) under inverse reuse q (Q16, 2^16 <= q < 2^26) to physical MiB
floor(y * 2^16 / q) (reading R22) with phys_div (estimate.cu): k = trunc(float(y) * (65536 / float(q))) with an
approximate reciprocal (__fdividef, <= 2 ulp), then one integer remainder test on each side. The claim: k is
within one of the quotient, so the corrected value is exact. Here the float estimate is modelled in float32 with
the reciprocal pushed 2 ulp either way (the device hook itself is pinned on the GPU:
tests/test_parity_gpu.py::test_exact_division_hook)."""
import numpy as np


def _phys_div_model(y, q, ulps):
    yf = y.astype(np.float32)
    qf = q.astype(np.float32)
    r = np.float32(65536.0) / qf
    for _ in range(abs(ulps)):
        r = np.nextafter(r, np.float32(np.inf if ulps > 0 else 0.0)).astype(np.float32)
    k = np.trunc(yf * r).astype(np.int64)
    rem = (y.astype(np.int64) << 16) - k * q.astype(np.int64)
    assert np.all(rem > -q.astype(np.int64)) and np.all(rem < 2 * q.astype(np.int64)), "estimate off by more than 1"
    return np.where(rem < 0, k - 1, np.where(rem >= q.astype(np.int64), k + 1, k))


def _check(y, q):
    y = np.asarray(y, np.uint64)
    q = np.asarray(q, np.uint64)
    want = ((y << np.uint64(16)) // q).astype(np.int64)
    for ulps in (-2, 0, 2):
        got = _phys_div_model(y, q, ulps)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (ulps, y[bad[:5]], q[bad[:5]])


def test_phys_div_random():
    rng = np.random.default_rng(2508)
    n = 2_000_000
    _check(rng.integers(0, 1 << 18, n), rng.integers(1 << 16, 1 << 26, n))
    _check(rng.integers(0, 1 << 18, n), rng.integers(1 << 16, 1 << 18, n))  # the generated regime


def test_phys_div_near_integer_quotients_and_edges():
    rng = np.random.default_rng(18556)
    y = rng.integers(1, 1 << 18, 1_000_000, dtype=np.uint64)
    k = rng.integers(1, 1 << 12, y.size, dtype=np.uint64)  # target quotient
    base = (y << np.uint64(16)) // k  # q' = base - 1, base, base + 1 put y * 2^16 / q' on or next to k
    for d in (0, 1, 2):
        _check(y, np.clip(base + np.uint64(d), (1 << 16) + 1, 1 << 26).astype(np.uint64) - np.uint64(1))
    j = rng.integers(16, 26, y.size).astype(np.uint64)  # exact quotients: q = 2^j
    _check(y, np.uint64(1) << j)
    ys = np.array([(1 << 18) - 1] * 4 + [0, 1, 2, 3, 65535, 65536], np.uint64)
    qs = np.array([1 << 16, (1 << 16) + 1, (1 << 26) - 1, (1 << 26) - 3, 1 << 16, 1 << 16, 65537, 196608, 65536,
                   65537], np.uint64)
    _check(ys, qs)
