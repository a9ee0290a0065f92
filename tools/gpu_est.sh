#!/bin/bash
# k_estimate check: GPU parity suite (or subset), configs 3 and 4 bench lines (kernel times), optional ncu of k_estimate.
# usage: gpurun -- 'bash tools/gpu_est.sh <tag> [pytest-args] [ncu]'
tag=${1:-est}
timeout 1500 python -m pytest tests -m gpu -x -q ${2:-} 2>&1 | tail -3
for c in 4 3; do
  echo -n "config $c: "
  timeout 300 python bench.py --no-cpu --no-e2e --config $c --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('%.3f ms/step' % d['ms_per_step'], 'est %.3f' % d['kernels']['k_estimate_ms'], {k: round(v,3) for k,v in d['kernels']['launch_ms'].items()}, r['bound'], 'alu frac %.3f' % r['alu']['frac'], 'it/s %.3e' % d.get('iteration_steps_per_s', 0))"
done
if [ "${3:-}" = "ncu" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_estimate -c 1 -o gpurun_out/${tag}_est_c4 -f \
    python bench.py --no-cpu --no-e2e --config 4 --steps 1 --warmup 0 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_est_c4.ncu-rep | grep -E "duration|inst_issued|inst_executed.sum|per_inst|dram__bytes"
fi
