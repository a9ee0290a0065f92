timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for v in "8 narrow" "8 wide" "32 narrow"; do set -- $v; MIG_LANES_PER_TRACE=$1 MIG_JOB_LAYOUT=$2 timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$v', d['value'], d['kernels'])"; done
timeout 300 python bench.py --no-cpu --no-e2e --config 5 --traces 2000000 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('c5', d['value'], d['kernels'])"
