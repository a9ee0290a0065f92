"""Alg. 1 on the device (mig_reachability: on-device reachability for larger state spaces),
against the host tables of the loaded geometries, the oracle's literal Alg. 1 (oracle.reach, itself pinned by the
pure-Python definition in tests/bruteforce.py) on random slot geometries, closed forms, and the invariants of Alg. 1
at 16-24 slots."""
import json
import time

import numpy as np
import pytest
import torch

import bruteforce as bf
from conftest import geom_path
from oracle import oracle as orc

import paper_2508_18556_b200 as mig

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["a30-24gb", "a100-40gb", "a100-80gb", "h100-80gb", "a100-40gb-1g10",
                                  "b200-180gb"])
def test_matches_loaded_geometry_tables(name):
    spec = json.load(open(geom_path(name)))
    n = spec["total_memory_slots"]
    fcr, flags, info = mig.mig_reachability(n, bf.geometry_masks(spec))
    g = mig.mig_geometry_load(f"builtin:{name}")
    host = np.array([mig.mig_geometry_fcr(g, m) for m in range(1 << n)], np.int64)
    dev = fcr.cpu().numpy().astype(np.int64)
    assert np.array_equal(dev, host)
    assert (info["n_states"], info["n_finals"], info["fcr_s0"]) == (g.info.n_states, g.info.n_finals, g.info.fcr_s0)
    fl = flags.cpu().numpy()
    assert np.array_equal((fl & 1) != 0, host > 0) and np.array_equal(dev[(fl & 2) != 0], np.ones(((fl & 2) != 0).sum()))


def test_random_geometries_equal_oracle():
    rng = np.random.default_rng(11)
    for trial in range(12):
        n = int(rng.integers(5, 12))
        masks = set()
        for _ in range(int(rng.integers(3, 3 * n))):
            L = int(rng.integers(1, min(n, 6) + 1))
            s = int(rng.integers(0, n - L + 1))
            masks.add(((1 << L) - 1) << s)
        masks = sorted(masks)
        ref, S, F = orc.reach(n, masks)  # the oracle's literal Alg. 1 (pinned on the CPU by the brute force)
        fcr, _, info = mig.mig_reachability(n, masks)
        assert np.array_equal(fcr.cpu().numpy().astype(np.int64), ref.astype(np.int64)), (n, masks)
        assert (info["n_states"], info["n_finals"], info["fcr_s0"]) == (S, F, int(ref[0]))


def _binary(n):
    return [((1 << L) - 1) << s for L in [1 << k for k in range(n.bit_length())] if L <= n for s in range(0, n, L)]


def test_binary_geometry_closed_forms():
    # aligned power-of-two slots: |S| = f(n) = f(n/2)^2 + 1 (f(1) = 2), |F| = fcr(s0) = g(n) = g(n/2)^2 + 1 (g(1) = 1)
    f, g = {1: 2}, {1: 1}
    for n in (2, 4, 8, 16):
        f[n], g[n] = f[n // 2] ** 2 + 1, g[n // 2] ** 2 + 1
    for n in (8, 16):
        fcr, flags, info = mig.mig_reachability(n, _binary(n))
        assert (info["n_states"], info["n_finals"], info["fcr_s0"]) == (f[n], g[n], g[n])
        assert int(fcr[(1 << n) - 1]) == 1


def test_24_slots_invariants_and_time():
    # a 24-slot geometry in the vendor shape (sizes 1, 2, 3 (on 4), 4, 6, 12, 24 slots at aligned starts): Alg. 1's
    # invariants on all 2^24 occupancies (fcr(final) = 1, fcr(s0) = |F|, fcr never grows along a placement)
    n = 24
    masks = sorted({((1 << L) - 1) << s for L, step in [(1, 1), (2, 2), (4, 4), (6, 6), (12, 12), (24, 24)]
                    for s in range(0, n - L + 1, step)} | {0b111 << s for s in range(0, n, 4)})
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fcr, flags, info = mig.mig_reachability(n, masks)
    dt = time.perf_counter() - t0
    f = fcr.cpu().numpy().astype(np.int64)
    fl = flags.cpu().numpy()
    assert info["fcr_s0"] == info["n_finals"] == f[0] and info["n_states"] >= info["n_finals"] > 1
    assert (f[(fl & 2) != 0] == 1).all() and (f[(fl & 1) == 0] == 0).all() and (f[(fl & 1) != 0] >= 1).all()
    rng = np.random.default_rng(3)
    states = np.nonzero(fl & 1)[0]
    for m in rng.choice(states, 2000):
        for q in masks:
            if (q & int(m)) == 0:
                assert f[int(m) | q] <= f[int(m)]
    print(f"mig_reachability 24 slots: {info} in {dt * 1e3:.1f} ms")


def test_invalid_arguments_and_capacity():
    with pytest.raises(mig.MigError):
        mig.mig_reachability(25, [1])
    with pytest.raises(mig.MigError):
        mig.mig_reachability(4, [1 << 5])
    # every pair of slots is a placement: the full occupancy has 23!! > 2^32 decompositions (perfect matchings)
    with pytest.raises(mig.MigError, match="MIG_E_CAPACITY"):
        mig.mig_reachability(24, [(1 << i) | (1 << j) for i in range(24) for j in range(i + 1, 24)])
