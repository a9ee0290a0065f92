"""Arithmetic claims the CUDA path relies on (DESIGN.md §6 k_estimate), checked exhaustively at the edges and on
random samples, on the CPU (numpy float64 division is IEEE correctly rounded, like __ddiv_rn).

scan_tail maps a requested MiB y (< 2^18) and an inverse reuse ratio q (Q16, 1 <= q < 2^26) to physical MiB
floor(y * 2^16 / q) (reading R22) as floor(double(y << 16) / double(q)): the numerator is below 2^34, so the rounding
error of the quotient (< quotient * 2^-53) stays below 1/q, the smallest distance from a non-integer quotient to the
next integer."""
import numpy as np


def _check(y, q):
    y = np.asarray(y, np.uint64)
    q = np.asarray(q, np.uint64)
    num = y << np.uint64(16)
    want = num // q
    got = np.floor(num.astype(np.float64) / q.astype(np.float64)).astype(np.uint64)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (y[bad[:5]], q[bad[:5]])


def test_double_floor_division_random():
    rng = np.random.default_rng(2508)
    n = 2_000_000
    _check(rng.integers(0, 1 << 18, n), rng.integers(1, 1 << 26, n))
    _check(rng.integers(0, 1 << 18, n), rng.integers(65536, 1 << 18, n))  # the generated regime (q >= 1.0)


def test_double_floor_division_near_integer_quotients():
    rng = np.random.default_rng(18556)
    y = rng.integers(1, 1 << 18, 1_000_000, dtype=np.uint64)
    num = y << np.uint64(16)
    k = rng.integers(1, 1 << 12, y.size, dtype=np.uint64)  # target quotient
    base = num // k  # num / q' lands on or next to k for q' = base - 1, base, base + 1
    for d in (0, 1, 2):
        qq = np.clip(base + np.uint64(d), 2, (1 << 26) - 1).astype(np.uint64) - np.uint64(1)
        _check(y, qq)
    # exact divisors of the numerator (integer quotients): q = 2^j and q = y * 2^j'
    j = rng.integers(0, 26, y.size).astype(np.uint64)
    _check(y, np.uint64(1) << j)
    small = y[y < (1 << 10)]
    _check(small, small << np.uint64(16))
    # largest numerators against the largest and smallest denominators
    ys = np.array([(1 << 18) - 1] * 6 + [1, 2, 3], np.uint64)
    qs = np.array([1, 2, 3, (1 << 26) - 1, (1 << 26) - 3, 65537, (1 << 26) - 1, 3, 7], np.uint64)
    _check(ys, qs)
