#!/bin/bash
# Timing-only A/B of build/var/*.so on one config (no oracle leg), interleaved repeats, concurrent and serialised
# policy launches. usage: gpurun -- 'bash tools/gpu_abtime.sh [config] [reps]'
c=${1:-2}
cp paper_2508_18556_b200/libmig.so /tmp/libmig_orig.so
for rep in $(seq ${2:-5}); do
  for v in build/var/*.so; do
    cp $v paper_2508_18556_b200/libmig.so
    for conc in 1 0; do
      echo -n "$(basename $v) c$c conc=$conc: "
      MIG_CONCURRENT_POLICIES=$conc timeout 600 python bench.py --no-e2e --no-dynamic --no-cpu --config $c 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.4f ms/step sim %.4f' % (d['ms_per_step'], d['kernels']['k_simulate_ms']), {k: round(v,4) for k,v in d['kernels']['launch_ms'].items()})"
    done
  done
done
cp /tmp/libmig_orig.so paper_2508_18556_b200/libmig.so
