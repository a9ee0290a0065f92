#!/bin/bash
# Quick iteration: lane-kernel parity, config-2 bench line, ncu full capture of the k_simulate launches.
tag=${1:-iter}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('%.3e'%d['value'], d['kernels'])"
bash tools/gpu_ncu.sh 2 $tag > /dev/null 2>&1; ls gpurun_out/$tag.ncu-rep
