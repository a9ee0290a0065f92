#!/bin/bash
# A/B of build/var/*.so on the config-2 bench (FF launch / step times), interleaved repeats, each variant first
# checked by a quick parity subset. usage: gpurun -- 'bash tools/gpu_ab2.sh [repeats] [bench-args]'
reps=${1:-2}
cp paper_2508_18556_b200/libmig.so /tmp/libmig_orig.so
for v in build/var/*.so; do
  cp $v paper_2508_18556_b200/libmig.so
  echo -n "$(basename $v) parity: "
  timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "generated_configs or ragged or config1" 2>&1 | tail -1
done
for rep in $(seq $reps); do
  for v in build/var/*.so; do
    cp $v paper_2508_18556_b200/libmig.so
    echo -n "$(basename $v): "
    timeout 300 python bench.py --no-cpu --no-e2e --no-dynamic ${2:-} 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.4e dec/s %.3f ms/step' % (d['value'], d['ms_per_step']), {k: round(v,4) for k,v in d['kernels']['launch_ms'].items()}, 'est', round(d['kernels']['k_estimate_ms'],4))"
  done
done
cp /tmp/libmig_orig.so paper_2508_18556_b200/libmig.so
