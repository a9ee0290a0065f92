"""Every k_simulate variant (one lane per trace: k_ff_lane / k_base_lane / k_sa_group + k_simulate_lane, or
k_simulate_lane alone; or a group of 8 | 32 lanes per trace with job
staging layout wide | narrow; policy launches on two streams (default) or serialised, MIG_CONCURRENT_POLICIES) is
parity-checked against the oracle. The variant is chosen per process from MIG_LANES_PER_TRACE / MIG_JOB_LAYOUT, so each runs in a
subprocess."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r'''
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import numpy as np
from test_parity_gpu import run_pair, assert_same, check_totals, random_tiny_traces, SPECS
from tracegen import tracegen as tg
import json
from conftest import geom_path
for cfg, n in [(2, 300), (3, 400), (4, 1500), (5, 200)]:
    jobs, ext, off = tg.generate_host(cfg, n)
    got, want, tot = run_pair(tg.CONFIG_GEOMETRY[cfg], jobs, ext, off, SPECS, seed=tg.seed_of(cfg))
    assert_same(got, want)
    check_totals(got, tot)
spec = json.load(open(geom_path("a100-40gb")))
jobs, ext, off = random_tiny_traces(np.random.default_rng(3), spec, 300, 60)
specs = SPECS + [dict(kind=3, flags=3)]
got, want, tot = run_pair("a100-40gb", jobs, ext, off, specs, seed=7, common=dict(ctx_mib=256, reconfig_ticks=100))
assert_same(got, want)
print("variant OK")
'''


@pytest.mark.parametrize("lanes,layout,conc,fast,order", [("1", "narrow", "1", "1", "1"), ("1", "narrow", "0", "1", "1"),
                                                          ("1", "narrow", "1", "0", "1"), ("1", "narrow", "1", "1", "2"),
                                                          ("1", "narrow", "1", "0", "2"), ("1", "narrow", "1", "1", "0"),
                                                          ("8", "wide", "1", "1", "1"), ("8", "narrow", "1", "1", "1"),
                                                          ("32", "wide", "1", "1", "1"), ("32", "narrow", "1", "1", "1")])
def test_variant_parity(lanes, layout, conc, fast, order):
    # fast = "0": the generic k_simulate_lane for FUSION_FISSION and BASELINE (MIG_FF_FAST=0) and Scheme A's grouping
    # pass inside the lane kernel (MIG_SA_PREGROUP=0) instead of k_ff_lane / k_base_lane / k_sa_group; order = "2":
    # the traces visited in trace_order.cu's order at every size (default "1": from 4096 traces), "0": trace order
    env = dict(os.environ, MIG_LANES_PER_TRACE=lanes, MIG_JOB_LAYOUT=layout, MIG_CONCURRENT_POLICIES=conc,
               MIG_FF_FAST=fast, MIG_SA_PREGROUP=fast, MIG_TRACE_ORDER=order)
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "variant OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
