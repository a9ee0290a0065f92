#!/bin/bash
# A/B the libmig builds in build/var/*.so on the config-2 bench (kernel times), after the parity suite.
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
cp paper_2508_18556_b200/libmig.so /tmp/libmig_orig.so
for v in build/var/*.so; do
  cp $v paper_2508_18556_b200/libmig.so
  for c in ${CONFIGS:-2}; do
    echo -n "$(basename $v) c$c: "
    timeout 300 python bench.py --no-cpu --no-e2e --config $c 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('%.3e'%d['value'], {k: (round(v,3) if isinstance(v,float) else v) for k,v in d['kernels'].items()})"
  done
done
cp /tmp/libmig_orig.so paper_2508_18556_b200/libmig.so
