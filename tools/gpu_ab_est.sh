#!/bin/bash
# A/B of build/var/*.so on configs 4 and 3 (k_estimate times), after a quick estimate-parity subset per variant.
cp paper_2508_18556_b200/libmig.so /tmp/libmig_orig.so
for v in build/var/*.so; do
  cp $v paper_2508_18556_b200/libmig.so
  echo -n "$(basename $v) parity: "
  timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "estimates or generated_configs or ewma or recorded" 2>&1 | tail -1
done
for rep in 1 2; do
  for v in build/var/*.so; do
    cp $v paper_2508_18556_b200/libmig.so
    for c in 4 3; do
      echo -n "$(basename $v) c$c: "
      timeout 300 python bench.py --no-cpu --no-e2e --config $c --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f ms/step' % d['ms_per_step'], 'est %.3f' % d['kernels']['k_estimate_ms'])"
    done
  done
done
cp /tmp/libmig_orig.so paper_2508_18556_b200/libmig.so
