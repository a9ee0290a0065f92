#!/bin/bash
# ncu --set full of one config-5 chunk's (4,194,304 traces) Scheme A launches: k_sa_group and the Scheme A lane
# kernel (k_simulate_lane<4, ...>), SASS source page of the lane kernel exported.
tag=${1:-sancu}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_sa_group|k_simulate_lane<.int.4" -c 2 \
  -o gpurun_out/$tag -f python bench.py --no-cpu --no-e2e --config 5 --traces 4194304 --steps 1 --warmup 0 > gpurun_out/$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep | grep -E "==|duration|inst_issued|inst_executed.sum|per_inst|dram__bytes|lts__t_bytes"
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source=sass --launch-skip 1 --launch-count 1 > gpurun_out/${tag}_src.csv 2>/dev/null
ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
rm -f gpurun_out/$tag.ncu-rep
