timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('%.3e'%d['value'], d['kernels'], d['roofline'])"
