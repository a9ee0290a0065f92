"""The multi-process oracle runner (oracle/pool.py) the full-size parity tests and bench.py use: it must give
exactly the single-process oracle's results and totals, and its element-by-element comparison must catch a
single differing field."""
import numpy as np

from conftest import geom_path
from oracle import oracle as orc
from oracle import pool
from tracegen import tracegen as tg

SPECS = [dict(kind=0), dict(kind=3), dict(kind=3, flags=1)]


def _direct(cfg, ids):
    g = orc.Geometry(geom_path(tg.CONFIG_GEOMETRY[cfg]))
    out = []
    for t in ids:
        j, e, o = tg.generate_host(cfg, 1, trace_id0=int(t))
        out.append(orc.simulate(g, j, e, o, [orc.policy(**s) for s in SPECS], seed=tg.seed_of(cfg),
                                trace_id0=int(t))[0])
    return np.stack(out)


def test_pool_range_and_ids_equal_direct(tmp_path):
    cfg = 3
    want = _direct(cfg, range(100, 160))
    r = pool.run(cfg, SPECS, t0=100, n=60, procs=3, want_results=True, block=7)
    assert np.array_equal(r["results"], want) and r["mismatches"] == 0 and r["traces"] == 60
    ids = np.arange(100, 160)[::-1].copy()
    r2 = pool.run(cfg, SPECS, ids=ids, procs=2, want_results=True, block=5)
    assert np.array_equal(r2["results"], want[::-1])
    tot = pool.totals_of(want)
    assert r["totals"] == tot and r2["totals"] == tot
    for p, t in enumerate(tot):
        assert t["n_traces"] == 60 and t["makespan_max"] == int(want[:, p]["makespan"].max())
        assert t["decision_hash_sum"] == int(sum(int(h) for h in want[:, p]["decision_hash"])) % 2**64
    # comparison mode: equal file -> 0 mismatches; one changed field in one row -> 1 mismatch, located
    path = str(tmp_path / "res.npy")
    np.save(path, want)
    assert pool.run(cfg, SPECS, t0=100, n=60, procs=2, cmp_path=path)["mismatches"] == 0
    bad = want.copy()
    bad[37, 2]["decision_hash"] ^= 1
    np.save(path, bad)
    r3 = pool.run(cfg, SPECS, t0=100, n=60, procs=2, cmp_path=path)
    assert r3["mismatches"] == 1 and r3["first"].startswith("trace 137 ") and "decision_hash" in r3["first"]
