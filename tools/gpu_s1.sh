#!/bin/bash
# Session start: parity suite, default bench line, SASS source pages of k_ff_lane (config 2) and k_estimate (config 4).
tag=${1:-s1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-e2e --cpu-seconds 5 --cpu-seconds-dynamic 3 > gpurun_out/${tag}_bench.json 2>gpurun_out/${tag}_bench.err; cut -c1-300 gpurun_out/${tag}_bench.json
bash tools/gpu_ffncu.sh ${tag}_ff
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_estimate -c 1 -o gpurun_out/${tag}_est -f \
  python bench.py --no-cpu --no-e2e --config 4 --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_est.ncu-rep | grep -E "duration|inst_issued|inst_executed.sum|per_inst|dram__bytes"
ncu -i gpurun_out/${tag}_est.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_est_src.csv 2>/dev/null
rm -f gpurun_out/${tag}_est.ncu-rep
