#!/bin/bash
# ncu --set full of k_ff_lane on config 2 (1M traces) with its SASS source page exported for tools/ncu_sass.py.
tag=${1:-ffncu}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ff_lane -c 1 -o gpurun_out/$tag -f \
  python bench.py --no-cpu --no-e2e --no-dynamic --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep | grep -E "duration|inst_issued|inst_executed.sum|per_inst|dram__bytes"
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_src.csv 2>/dev/null
rm -f gpurun_out/$tag.ncu-rep
