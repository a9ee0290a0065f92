#!/bin/bash
# A/B of build/var/*.so on k_estimate: estimate parity tests per variant, then configs 4 and 3 bench lines
# (k_estimate ms, the line's oracle parity), repeated interleaved. usage: gpurun -- 'bash tools/gpu_abest.sh [reps]'
cp paper_2508_18556_b200/libmig.so /tmp/libmig_orig.so
for v in build/var/*.so; do
  cp $v paper_2508_18556_b200/libmig.so
  echo "$(basename $v) tests: $(timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k 'estimates or generated_configs or recorded_samples or ewma or random_ragged' 2>&1 | tail -1)"
done
for rep in $(seq ${1:-2}); do
  for v in build/var/*.so; do
    cp $v paper_2508_18556_b200/libmig.so
    for c in 4 3; do
      echo -n "$(basename $v) c$c: "
      timeout 600 python bench.py --no-e2e --no-dynamic --config $c --steps 5 --cpu-seconds 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); p=d.get('parity',{}); r=d['roofline']; print('%.3f ms/step est %.3f sim %.3f' % (d['ms_per_step'], d['kernels']['k_estimate_ms'], d['kernels']['k_simulate_ms']), r['kernel'], 'alu %.4f' % r['alu']['frac'], 'parity', p.get('rows_checked'), p.get('rows_mismatched'))"
    done
  done
done
cp /tmp/libmig_orig.so paper_2508_18556_b200/libmig.so
