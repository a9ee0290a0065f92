#!/bin/bash
# Timing of the config-2 step under side-stream launch knobs (MIG_SIDE_FIRST, MIG_SIDE_CTAS) for build/var/*.so.
cp paper_2508_18556_b200/libmig.so /tmp/libmig_orig.so
for rep in 1 2; do
  for v in build/var/*.so; do
    cp $v paper_2508_18556_b200/libmig.so
    for knob in "0 0" "1 1" "1 2" "0 7"; do
      set -- $knob
      echo -n "$(basename $v) first=$1 ctas=$2: "
      MIG_SIDE_FIRST=$1 MIG_SIDE_CTAS=$2 timeout 600 python bench.py --no-e2e --no-dynamic --no-cpu --config ${C:-2} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.4f ms/step sim %.4f' % (d['ms_per_step'], d['kernels']['k_simulate_ms']), {k: round(v,4) for k,v in d['kernels']['launch_ms'].items()})"
    done
  done
done
cp /tmp/libmig_orig.so paper_2508_18556_b200/libmig.so
