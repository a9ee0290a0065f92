timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
MIG_LANES_PER_TRACE=32 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-900
MIG_LANES_PER_TRACE=32 timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-900
timeout 300 python bench.py --no-cpu --no-e2e --config 4 2>&1 | tail -1 | cut -c1-900
