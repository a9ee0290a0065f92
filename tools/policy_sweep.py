"""Policy sweep on the synthetic configs through the library (one GPU): for every policy, throughput and energy
relative to the non-partitioned BASELINE (the paper's normalisation), memory utilisation
(PAPER.md:675), OOMs, early restarts and wasted time. Writes a markdown table.

Usage: python tools/policy_sweep.py [--traces N] [--out profiles/r01_policy_sweep.md]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2508_18556_b200 as mig  # noqa: E402
from tracegen import tracegen as tg  # noqa: E402

NAMES = {0: "BASELINE", 1: "STATIC", 2: "DYNAMIC", 3: "FUSION_FISSION", 4: "SCHEME_A"}
POLICIES = [(0, 0), (1, 0), (2, 0), (3, 0), (3, 1), (4, 0), (4, 1)]


def sweep(cfg, n):
    geo = tg.CONFIG_GEOMETRY[cfg]
    g = mig.mig_geometry_load(f"builtin:{geo}")
    pols = []
    for k, f in POLICIES:
        if k == 1 and g.info.n_layout == 0:
            continue
        pols.append((k, f, mig.policy(g, kind=k, flags=f)))
    jobs, ext, off = tg.generate_device(cfg, n)
    tr = mig.Traces(jobs, ext, off, n, seed=tg.seed_of(cfg), max_jobs=tg.jobs_per_trace(cfg))
    _, tot = mig.mig_simulate(g, tr, [p for _, _, p in pols], write_results=False)
    torch.cuda.synchronize()
    t = mig.totals_numpy(tot)
    base = t[0]
    full_mib = g.info.full_mem_mib
    rows = []
    for i, (k, f, _) in enumerate(pols):
        r = t[i]
        # jobs completed per tick of makespan, and energy per completed job, relative to BASELINE
        thr = (float(r["completed"]) / float(r["makespan_sum"])) / (float(base["completed"]) / float(base["makespan_sum"]))
        en = (float(base["energy_wticks"]) / float(base["completed"])) / (float(r["energy_wticks"]) / float(r["completed"]))
        util = float(r["mem_mib_ticks"]) / (full_mib * float(r["makespan_sum"]))
        name = NAMES[k] + ("+ER" if f & 1 else "")
        rows.append((name, thr, en, util, int(r["completed"]), int(r["rejected"]), int(r["ooms"]),
                     int(r["preempts"]), float(r["wasted_ticks"]) / max(1, int(r["n_traces"])),
                     int(r["placements"]) + int(r["waits"]) + int(r["rejected"])))
    return geo, rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traces", type=int, default=100_000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_policy_sweep.md"))
    a = ap.parse_args()
    lines = ["# Policy sweep on the synthetic configs (one B200, `tools/policy_sweep.py`)", "",
             f"{a.traces} traces per config. Throughput (completed jobs per tick of makespan) and energy per completed job "
             "are relative to BASELINE (the non-partitioned GPU, PAPER.md:635-637), > 1 is better. Memory utilisation = MiB-ticks / "
             "(GPU MiB x makespan) (PAPER.md:675). These are synthetic workloads shaped like the paper's; the paper's "
             "own ratios (6.20x / 5.93x general, 1.59x / 1.12x ML, 1.43x / 1.11x LLM on an A100) are context only.",
             ""]
    for cfg in (2, 3, 4, 5):
        geo, rows = sweep(cfg, a.traces)
        lines += [f"## Config {cfg} ({geo})", "",
                  "| policy | throughput x | energy x | memory util | completed | rejected | OOMs | early restarts | "
                  "wasted ticks / trace | decisions |",
                  "|---|---|---|---|---|---|---|---|---|---|"]
        for r in rows:
            lines.append(f"| {r[0]} | {r[1]:.2f} | {r[2]:.2f} | {r[3]:.3f} | {r[4]} | {r[5]} | {r[6]} | {r[7]} | "
                         f"{r[8]:.0f} | {r[9]} |")
        lines.append("")
    text = "\n".join(lines)
    with open(a.out, "w") as f:
        f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
