#!/bin/bash
# One gpurun call: GPU parity suite, smoke, default bench line, ncu launch list of the bench step.
# usage: gpurun --timeout 2400 -- 'bash tools/gpu_check.sh <tag>'
tag=${1:-check}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -3 gpurun_out/bench_$tag.err
cut -c1-1500 gpurun_out/bench_$tag.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > /dev/null 2>&1
echo "launches: $(wc -l < gpurun_out/launches_$tag.csv)"
