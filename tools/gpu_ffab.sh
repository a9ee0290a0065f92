#!/bin/bash
# Parity (GPU suite or a subset), A/B of the config-2 bench (MIG_FF_FAST=1 k_ff_lane vs 0 k_simulate_lane<FF>),
# then an ncu --set full capture of k_ff_lane with its key metrics.
# usage: gpurun -- 'bash tools/gpu_ffab.sh <tag> [pytest-args]'
tag=${1:-ff}
timeout 1500 python -m pytest tests -m gpu -x -q ${2:-} 2>&1 | tail -4
for rep in 1 2; do
  for v in 1 0; do
    echo -n "MIG_FF_FAST=$v: "
    MIG_FF_FAST=$v timeout 300 python bench.py --no-cpu --no-e2e --no-dynamic 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.4e dec/s %.3f ms/step' % (d['value'], d['ms_per_step']), {k: round(v,4) for k,v in d['kernels']['launch_ms'].items()}, 'est', round(d['kernels']['k_estimate_ms'],4))"
  done
done
bash tools/gpu_ncu.sh 2 $tag regex:k_ff_lane > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep | grep -E "duration|inst_issued|inst_executed.sum|per_inst|dram__bytes"
