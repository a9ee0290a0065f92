#!/bin/bash
# Scheme A pre-grouping A/B: parity suite subset, then config 5 (one 2^22-trace chunk, resident) with
# MIG_SA_PREGROUP=1 / 0: per-launch times.
timeout 1500 python -m pytest tests -m gpu -x -q ${1:-tests/test_parity_gpu.py tests/test_kernel_variants_gpu.py} 2>&1 | tail -3
for rep in 1 2; do
  for v in 1 0; do
    echo -n "MIG_SA_PREGROUP=$v: "
    MIG_SA_PREGROUP=$v timeout 600 python bench.py --no-cpu --no-e2e --config 5 --traces 4194304 --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f ms/step' % d['ms_per_step'], {k: round(v,3) for k,v in d['kernels']['launch_ms'].items()}, 'est', round(d['kernels']['k_estimate_ms'],3))"
  done
done
