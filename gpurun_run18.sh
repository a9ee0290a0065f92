timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
for c in 2 4; do timeout 300 python bench.py --no-cpu --no-e2e --config $c 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('config $c', '%.3e'%d['value'], d['kernels'])"; done
