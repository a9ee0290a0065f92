timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for L in 1 8; do MIG_LANES_PER_TRACE=$L timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('lanes $L', '%.3e'%d['value'], d['kernels'])"; done
for c in 3 4 5; do timeout 300 python bench.py --no-cpu --no-e2e --config $c 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('config $c', '%.3e'%d['value'], d['kernels'])"; done
