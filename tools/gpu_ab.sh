#!/bin/bash
# A/B the libmig builds in build/var/*.so on the config-2 bench (kernel times, 3 repeats each, interleaved),
# after the parity suite on the in-tree build. usage: gpurun -- 'bash tools/gpu_ab.sh [configs]'
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
cp paper_2508_18556_b200/libmig.so /tmp/libmig_orig.so
for rep in 1 2 3; do
  for v in build/var/*.so; do
    cp $v paper_2508_18556_b200/libmig.so
    for c in ${1:-2}; do
      echo -n "$(basename $v) c$c: "
      timeout 300 python bench.py --no-cpu --no-e2e --config $c 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('%.4e'%d['value'], {k: (round(v,4) if isinstance(v,float) else ({a: round(b,4) for a,b in v.items()} if isinstance(v, dict) else v)) for k,v in d['kernels'].items()})"
    done
  done
done
cp /tmp/libmig_orig.so paper_2508_18556_b200/libmig.so
