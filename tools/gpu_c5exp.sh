#!/bin/bash
# Experiment runner: bench kernel times for env / build variants (edit per experiment).
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
run() { echo -n "$1 $2 c$3: "; cp build/var/$2 paper_2508_18556_b200/libmig.so; env $1 timeout 300 python bench.py --no-cpu --no-e2e --config $3 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('%.4e'%d['value'], round(d['kernels']['k_simulate_ms'],3), {a: round(b,3) for a,b in d['kernels']['launch_ms'].items()})"; }
for rep in 1 2; do
for c in 2 5; do
run "X=1" c_conc.so $c
run "X=1" d_l1.so $c
run "MIG_CARVEOUT=72" d_l1.so $c
run "MIG_CARVEOUT=58" d_l1.so $c
done
done
cp build/var/d_l1.so paper_2508_18556_b200/libmig.so
