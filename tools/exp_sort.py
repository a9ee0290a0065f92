"""Experiment: does ordering config-2 traces by a similarity signature (the tight-fit levels of the first jobs and
whether their iteration times agree) make the lanes of a k_ff_lane warp share phases? Times mig_simulate on the
generated order and on the sorted order (same traces, per-policy totals must be equal)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_18556_b200 as mig  # noqa: E402
from tracegen import tracegen as tg  # noqa: E402

dev = torch.device("cuda", 0)
cfg, n = 2, 1_000_000
J = tg.jobs_per_trace(cfg)
jobs, ext, off = tg.generate_device(cfg, n, seed=tg.seed_of(cfg), device=dev)
g = mig.mig_geometry_load("builtin:a100-40gb")
levels = torch.tensor([5120, 10240, 20480, 40960], device=dev, dtype=torch.int64)
j3 = jobs.view(n, J, 4).to(torch.int64)
need = torch.searchsorted(levels, (j3[:, :, 0] & 0xFFFFFFFF) + 512)  # level of each job's tight fit
K = int(os.environ.get("SIG_JOBS", "4"))
mode = os.environ.get("SIG_MODE", "levels")
same_t = (j3[:, :K, 3] == j3[:, :1, 3]).all(dim=1).to(torch.int64)
key = same_t
for k in range(K):
    key = key * 8 + need[:, k]
if mode in ("oom", "oom_homog"):  # + the position of the first job whose estimate is below its true footprint
    under = (j3[:, :, 0] & 0xFFFFFFFF) < (j3[:, :, 1] & 0xFFFFFFFF)
    first = torch.where(under.any(dim=1), under.to(torch.int64).argmax(dim=1), torch.full_like(key, J))
    key = key * 128 + first
if mode == "oom_homog":  # + all jobs of one level and one iteration time
    homog = ((need == need[:, :1]).all(dim=1) & (j3[:, :, 3] == j3[:, :1, 3]).all(dim=1)).to(torch.int64)
    key = homog * (1 << 40) + key
if mode in ("ticks", "ticks2"):  # + the octave of the first job's (jobs') iteration time
    for k in range(1 if mode == "ticks" else 2):
        lt = torch.floor(torch.log2(j3[:, k, 3].clamp(min=1).to(torch.float64))).to(torch.int64).clamp(0, 15)
        key = key * 16 + lt
if os.environ.get("SIG_DESC"):
    key = -key
perm = torch.argsort(key, stable=True)
jobs_s = jobs.view(n, J, 4)[perm].reshape(-1, 4).contiguous()


def run(jb, label, pols, reps=20):
    tr = mig.Traces(jb, None, off, n, seed=tg.seed_of(cfg), max_jobs=J, flags=mig.MIG_TRACES_NO_DYNAMIC)
    res = torch.empty((n * len(pols), 96), dtype=torch.uint8, device=dev)
    tot = torch.empty((len(pols), 192), dtype=torch.uint8, device=dev)
    for _ in range(3):
        mig.mig_simulate(g, tr, pols, out=res, totals=tot)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        mig.mig_simulate(g, tr, pols, out=res, totals=tot)
    b.record()
    torch.cuda.synchronize()
    print(f"{label}: {a.elapsed_time(b) / reps:.4f} ms/step", flush=True)
    return mig.totals_numpy(tot)


for pols, name in [([mig.policy(g, kind=3)], "FF"), ([mig.policy(g, kind=3), mig.policy(g, kind=0)], "FF+BASE")]:
    t0 = run(jobs, f"{name} generated order", pols)
    t1 = run(jobs_s, f"{name} sorted (K={K}, {mode})", pols)
    assert all((t0[f] == t1[f]).all() for f in t0.dtype.names), "totals differ"
print("classes:", int(torch.unique(key).numel()))
