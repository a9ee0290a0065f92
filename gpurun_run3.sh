timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -2
