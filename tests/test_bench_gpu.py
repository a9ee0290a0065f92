"""bench.py's JSON contract on a small run (the driver parses this line): one line on stdout with the metric and
config BASELINE.json names, the timing keys, roofline, cpu_baseline, e2e, gpu_launches and clocks; and the
reference arm (the CPU oracle) in the same shape."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _run(args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_keys():
    d = _run(["--steps", "3", "--warmup", "3", "--traces", "20000", "--dynamic-traces", "20000", "--cpu-seconds", "1",
              "--cpu-seconds-dynamic", "1", "--e2e-steps", "1"])
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert d["metric"] == json.load(f)["metric"]
    for k in ["value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "vs_baseline",
              "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks", "parity",
              "dynamic_path"]:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["unit"] == "decisions/s" and d["config"]["workload"].startswith("config2")
    # per step: one lane launch per policy (MIG_TRACES_NO_DYNAMIC: no estimator) + the visit-order pass (3 launches;
    # config 2's 100-job queues, 20000 traces)
    assert d["gpu_launches"] == 3 * (2 + 3)
    r = d["roofline"]
    assert r["bound"] in ("hbm", "alu") and 0 < r["frac"] < 1 and r["achieved"] > 0 and r["peak"] > 0
    assert r["frac"] == (r["hbm"]["frac"] if r["bound"] == "hbm" else r["alu"]["frac"])
    assert (r["intensity_ops_per_byte"] < r["ridge_ops_per_byte"]) == (r["bound"] == "hbm")
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    p = d["parity"]
    assert p["rows_mismatched"] == 0 and p["traces_checked"] > 0
    if p["mode"] == "full":
        assert p["totals_equal"] is True and p["traces_checked"] == 20000
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    dp = d["dynamic_path"]
    assert dp["workload"].startswith("config4") and dp["value"] > 0 and dp["parity"]["rows_mismatched"] == 0
    assert dp["roofline"]["kernel"] == "k_estimate" and dp["early_restart"]["preempts"] > 0


def test_bench_chunked_strong_scaling():
    # config 5 path at reduced size: 3 x 10^5 traces over "all GPUs" (strong), generated in chunks of 10^5 inside
    # the step; the oracle samples the GPU's ids
    d = _run(["--config", "5", "--total-traces", "300000", "--chunk", "100000", "--steps", "3", "--warmup", "3",
              "--cpu-seconds", "1", "--no-e2e"])
    assert d["scaling"] == "strong" and d["config"]["total_traces"] == 300000
    assert d["gpu_launches"] == 3 * 3 * 7  # per step: 3 chunks x (k_estimate + 6 policies)
    assert d["parity"]["rows_mismatched"] == 0 and d["value"] > 0
