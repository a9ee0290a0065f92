#!/bin/bash
# ncu --set full of the Scheme A lane launch on one config-5 chunk (4,194,304 traces), SASS source page exported.
tag=${1:-sancu}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_simulate_lane --launch-skip 5 -c 1 \
  -o gpurun_out/$tag -f python bench.py --no-cpu --no-e2e --config 5 --traces 4194304 --steps 1 --warmup 0 > gpurun_out/$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep | grep -E "==|duration|inst_issued|inst_executed.sum|per_inst|dram__bytes"
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_src.csv 2>/dev/null
rm -f gpurun_out/$tag.ncu-rep
