#!/bin/bash
# A/B of the libmig builds in build/var/*.so on config 2: per variant, the fast-kernel parity tests and the bench
# line (oracle re-simulation of every trace: parity rows_mismatched), repeated interleaved.
# usage: gpurun -- 'bash tools/gpu_abff.sh [reps] [pytest -k expr] [bench args]'
reps=${1:-2}
kexpr=${2:-"fast_kernels or config1 or generated_configs or random_ragged or max_length"}
cp paper_2508_18556_b200/libmig.so /tmp/libmig_orig.so
for v in build/var/*.so; do
  cp $v paper_2508_18556_b200/libmig.so
  echo "$(basename $v) tests: $(timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "$kexpr" 2>&1 | tail -1)"
done
for rep in $(seq $reps); do
  for v in build/var/*.so; do
    cp $v paper_2508_18556_b200/libmig.so
    echo -n "$(basename $v): "
    timeout 300 python bench.py --no-e2e --no-dynamic --cpu-seconds 8 ${3:-} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); p=d.get('parity',{}); print('%.4e dec/s %.4f ms/step' % (d['value'], d['ms_per_step']), {k: round(v,4) for k,v in d['kernels']['launch_ms'].items()}, 'parity', p.get('mode'), p.get('rows_mismatched'), p.get('totals_equal'))"
  done
done
cp /tmp/libmig_orig.so paper_2508_18556_b200/libmig.so
