#!/bin/bash
# ncu --set full (+source) of the config-2 k_simulate launches and per-line listings; configs 3-4 bench lines.
# usage: gpurun --timeout 1800 -- 'bash tools/gpu_prof.sh <tag>'
tag=${1:-prof}
mkdir -p gpurun_out
bash tools/gpu_ncu.sh 2 $tag > /dev/null 2>&1
python tools/ncu_lines.py gpurun_out/$tag.ncu-rep 400 > gpurun_out/${tag}_lines.txt 2>&1
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep > gpurun_out/${tag}_summary.txt 2>&1
head -5 gpurun_out/${tag}_lines.txt
for c in 3 4; do timeout 600 python bench.py --no-cpu --no-e2e --config $c > gpurun_out/bench_${tag}_c$c.json 2>/dev/null; cut -c1-600 gpurun_out/bench_${tag}_c$c.json; done
