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


def _wrap64(v):
    """Two's-complement int64 wrap of a Python integer (what the device's int64 arithmetic yields)."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= 1 << 63 else v


def _ssr_int64_terms(y):
    """The first chunk's residual sum (n <= 32) formed term by term in wrapping int64, as k_estimate's fit_at does
    when n32 holds, next to the exact value: (n^2-1)(n Syy - Sy^2) - 3 Ky^2, Ky = 2 Sty - (n+1) Sy."""
    out = []
    Sy = Sty = Syy = 0
    for i, v in enumerate(y, 1):
        Sy += v
        Sty += i * v
        Syy += v * v
        n = i
        Ky = 2 * Sty - (n + 1) * Sy
        exact = (n * n - 1) * (n * Syy - Sy * Sy) - 3 * Ky * Ky
        a = _wrap64(n * Syy - Sy * Sy)
        b = _wrap64((n * n - 1) * a)
        c = _wrap64(3 * _wrap64(Ky * Ky))
        out.append((exact, _wrap64(b - c)))
    return out


def test_first_chunk_residual_sum_fits_int64():
    # estimate.cu fit_at(n32): for n <= 32 and samples y < 2^18 every term of the residual sum stays below 2^60, so
    # the int64 evaluation equals the exact (int128) one. Edges: constant maximum, alternating 0 / maximum, ramps, and
    # random series at the bound.
    top = (1 << 18) - 1
    series = [[top] * 32, [0, top] * 16, [top, 0] * 16, list(range(top - 31, top + 1)), [top - 40 * i for i in range(32)],
              [0] * 31 + [top], [top] + [0] * 31]
    rng = np.random.default_rng(7)
    series += [list(rng.integers(0, 1 << 18, 32)) for _ in range(2000)]
    series += [list(rng.integers(top - 64, 1 << 18, 32)) for _ in range(500)]
    for y in series:
        for exact, got in _ssr_int64_terms([int(v) for v in y]):
            assert got == exact and abs(exact) < 1 << 61
