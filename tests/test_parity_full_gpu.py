"""Full-size parity at SURVEY.md §8(d)'s coverage, in bench.py's launch configuration (device-generated traces, all
policies in one mig_simulate call per batch):

  C2, C3  every one of the 10^6 traces x 7 policies, element by element against the oracle;
  C4      10^7 traces on the device, every 10th (10^6) against the oracle;
  C5      10^8 traces generated and simulated on one GPU in chunks of 2^22 (sharding.simulate_generated), every
          1000th (10^5) against the oracle.

The oracle runs on every host core (oracle/pool.py: one process per core, each regenerating its traces on the
host and comparing its rows of the device's results). Besides every (trace, policy) row, the per-policy totals of
the device (decision-hash sum included) must equal the oracle's bit for bit wherever the oracle covers the launch.
"""
import os

import numpy as np
import pytest
import torch

from oracle import pool
from tracegen import tracegen as tg

import paper_2508_18556_b200 as mig
from paper_2508_18556_b200.sharding import simulate_generated

pytestmark = pytest.mark.gpu

SPECS = [dict(kind=0), dict(kind=1), dict(kind=2), dict(kind=3), dict(kind=3, flags=1), dict(kind=4),
         dict(kind=4, flags=1)]


def _device_run(cfg, n):
    g = mig.mig_geometry_load(f"builtin:{tg.CONFIG_GEOMETRY[cfg]}")
    seed = tg.seed_of(cfg)
    dj, de, do = tg.generate_device(cfg, n)
    tr = mig.Traces(dj, de, do, n, seed=seed, max_jobs=tg.jobs_per_trace(cfg))
    pols = [mig.policy(g, **s) for s in SPECS]
    res, tot = mig.mig_simulate(g, tr, pols)
    torch.cuda.synchronize()
    del dj, de, do, tr
    return res, mig.totals_numpy(tot)


def _assert_totals_equal(dev_tot, orc_tot):
    for p, (d, o) in enumerate(zip(dev_tot, orc_tot)):
        for f in pool.TOTALS_FIELDS:
            assert int(d[f]) == o[f], (SPECS[p], f, int(d[f]), o[f])


def _save(tmp_path, rows):
    path = os.path.join(str(tmp_path), "dev_results.npy")
    np.save(path, rows)
    return path


@pytest.mark.parametrize("cfg", [2, 3])
def test_full_parity_every_trace(cfg, tmp_path):
    n = tg.CONFIG_TRACES[cfg]
    res, dev_tot = _device_run(cfg, n)
    rows = mig.results_numpy(res, len(SPECS))
    del res
    r = pool.run(cfg, SPECS, t0=0, n=n, cmp_path=_save(tmp_path, rows))
    assert r["mismatches"] == 0, f"{r['mismatches']} (trace, policy) rows differ; first: {r['first']}"
    assert r["traces"] == n
    _assert_totals_equal(dev_tot, r["totals"])  # the whole launch: every field, decision_hash_sum included


def test_config4_stride10(tmp_path):
    cfg, n, stride = 4, tg.CONFIG_TRACES[4], 10
    res, dev_tot = _device_run(cfg, n)
    ids = np.arange(0, n, stride, dtype=np.int64)
    sel = res.view(n, len(SPECS), 96)[torch.from_numpy(ids).to(res.device)]
    rows = sel.cpu().numpy().view(mig.RESULT_DTYPE).reshape(-1, len(SPECS))
    del res, sel
    r = pool.run(cfg, SPECS, ids=ids, cmp_path=_save(tmp_path, rows), block=2048)
    assert r["mismatches"] == 0, f"{r['mismatches']} (trace, policy) rows differ; first: {r['first']}"
    assert r["traces"] == n // stride
    assert all(int(t["n_traces"]) == n and int(t["error_flags"]) == 0 for t in dev_tot)


def test_config5_1e8_chunked_stride1000(tmp_path):
    cfg, n, stride = 5, tg.CONFIG_TRACES[5], 1000
    g = mig.mig_geometry_load(f"builtin:{tg.CONFIG_GEOMETRY[cfg]}")
    pols = [mig.policy(g, **s) for s in SPECS]
    tot, smp = simulate_generated(g, cfg, pols, 0, n, chunk=1 << 22, sample_stride=stride)
    torch.cuda.synchronize()
    rows = smp.cpu().numpy().view(mig.RESULT_DTYPE).reshape(-1, len(SPECS))
    ids = np.arange(0, n, stride, dtype=np.int64)
    assert len(rows) == len(ids)
    r = pool.run(cfg, SPECS, ids=ids, cmp_path=_save(tmp_path, rows), block=1024)
    assert r["mismatches"] == 0, f"{r['mismatches']} (trace, policy) rows differ; first: {r['first']}"
    t = tot.cpu().numpy()
    assert (t[:, 0] == n).all() and (t[:, 20] == 0).all()  # every trace simulated, no format errors
    # the sample's totals, recomputed from the device rows, equal the oracle's
    assert pool.totals_of(rows) == r["totals"]


def test_chunked_equals_unchunked():
    # the chunk loop is transparent: 2^20 traces of config 5 in chunks of 3 x 10^5 (ragged last chunk) give the
    # totals and the sampled rows of one launch over all of them
    cfg, n, stride = 5, 1 << 20, 97
    g = mig.mig_geometry_load(f"builtin:{tg.CONFIG_GEOMETRY[cfg]}")
    pols = [mig.policy(g, **s) for s in SPECS]
    t_a, s_a = simulate_generated(g, cfg, pols, 5_000_000, n, chunk=300_000, sample_stride=stride)
    t_b, s_b = simulate_generated(g, cfg, pols, 5_000_000, n, chunk=n, sample_stride=stride)
    torch.cuda.synchronize()
    assert torch.equal(t_a, t_b) and torch.equal(s_a, s_b)
    assert int(t_a[0, 0]) == n
