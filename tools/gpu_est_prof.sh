#!/bin/bash
# ncu --set full (+source) of k_estimate on config 4 (2M traces) and its per-line listing.
tag=${1:-est}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_estimate -c 1 \
  -o gpurun_out/$tag -f python bench.py --no-cpu --no-e2e --config 4 --traces 2000000 --steps 1 --warmup 0 > gpurun_out/$tag.log 2>&1
python tools/ncu_lines.py gpurun_out/$tag.ncu-rep 120 > gpurun_out/${tag}_lines.txt 2>&1
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep > gpurun_out/${tag}_summary.txt 2>&1
head -3 gpurun_out/${tag}_lines.txt
