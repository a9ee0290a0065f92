import sys, json
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
from test_parity_gpu import random_tiny_traces, random_arrivals, run_pair
from conftest import geom_path
from oracle import oracle as orc
from tracegen import tracegen as tg
geo = "a30-24gb"
spec = json.load(open(geom_path(geo)))
rng = np.random.default_rng(31)
jobs, ext, off = random_tiny_traces(rng, spec, 600, 30, xfer=True)
arrival = random_arrivals(rng, off, 3000)
t = 9
a, b = int(off[t]), int(off[t+1])
J, E, O, A = jobs[a:b], ext[a:b], np.array([0, b-a], np.uint64), arrival[a:b]
print("jobs", b-a, "arrivals", A.tolist())
for kind in [1, 2, 3]:
    got, want, tot = run_pair(geo, J, E, O, [dict(kind=kind)], seed=37, common=dict(ctx_mib=0, reconfig_ticks=0), arrival=A)
    print(kind, "gpu", {f: int(got[f][0,0]) for f in ["makespan","placements","waits","rejected","ooms","completed","turnaround_sum"]})
    print(kind, "orc", {f: int(want[f][0,0]) for f in ["makespan","placements","waits","rejected","ooms","completed","turnaround_sum"]})
og = orc.Geometry(geom_path(geo))
r, recs = orc.simulate(og, J, E, O, orc.policy(kind=1, ctx_mib=0, reconfig_ticks=0), seed=37, records=True, arrival=A, trace_id0=0)
for x in recs: print(x)
for j in range(b-a): print(j, [int(v) for v in J[j]], [int(v) for v in E[j]], int(A[j]))
