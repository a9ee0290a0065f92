#!/bin/bash
# Fast kernels with extension records / early restart: GPU parity suite, then configs 3/4 (and 2) bench lines with
# MIG_FF_FAST=1 (k_ff_lane / k_base_lane) vs 0 (k_simulate_lane) — kernel times and the lines' oracle parity.
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 3 4 2; do
  for v in 1 0; do
    echo -n "config $c MIG_FF_FAST=$v: "
    MIG_FF_FAST=$v timeout 600 python bench.py --no-e2e --no-dynamic --config $c --steps 10 --cpu-seconds 8 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); p=d.get('parity',{}); print('%.3f ms/step' % d['ms_per_step'], {k: round(v,3) for k,v in d['kernels']['launch_ms'].items()}, 'est %.2f sim %.2f' % (d['kernels']['k_estimate_ms'], d['kernels']['k_simulate_ms']), 'parity', p.get('mode'), p.get('rows_checked'), p.get('rows_mismatched'), p.get('totals_equal'))"
  done
done
