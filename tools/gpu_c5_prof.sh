#!/bin/bash
# ncu --set full (+source) of config 5's Scheme A lane launch (the 6th k_simulate_lane launch; 2M traces).
tag=${1:-c5prof}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_simulate_lane -s 5 -c 1 \
  -o gpurun_out/$tag -f python bench.py --no-cpu --no-e2e --config 5 --traces 2000000 --steps 1 --warmup 0 > gpurun_out/$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep > gpurun_out/${tag}_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/$tag.ncu-rep 80 > gpurun_out/${tag}_lines.txt 2>&1
tail -2 gpurun_out/$tag.log | cut -c1-200
