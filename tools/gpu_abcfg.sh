#!/bin/bash
# A/B of build/var/*.so over configs: per variant the lane-kernel parity tests, then per config the bench line (step,
# k_estimate, k_simulate, per-launch ms, the line's oracle parity), repeated interleaved.
# usage: gpurun -- 'bash tools/gpu_abcfg.sh "<configs>" [reps] [pytest -k]'
cfgs=${1:-"2 4"}
kexpr=${3:-"fast_kernels or config1 or generated_configs or random_ragged or max_length or arrival or pcie"}
cp paper_2508_18556_b200/libmig.so /tmp/libmig_orig.so
for v in build/var/*.so; do
  cp $v paper_2508_18556_b200/libmig.so
  echo "$(basename $v) tests: $(timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "$kexpr" 2>&1 | tail -1)"
done
for rep in $(seq ${2:-2}); do
  for v in build/var/*.so; do
    cp $v paper_2508_18556_b200/libmig.so
    for c in $cfgs; do
      st=20; [ $c = 5 ] && st=2
      echo -n "$(basename $v) c$c: "
      timeout 900 python bench.py --no-e2e --no-dynamic --config $c --steps $st --cpu-seconds 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); p=d.get('parity',{}); print('%.3f ms/step est %.3f sim %.3f' % (d['ms_per_step'], d['kernels']['k_estimate_ms'], d['kernels']['k_simulate_ms']), {k: round(v,3) for k,v in d['kernels']['launch_ms'].items()}, 'parity', p.get('rows_checked'), p.get('rows_mismatched'))"
    done
  done
done
cp /tmp/libmig_orig.so paper_2508_18556_b200/libmig.so
