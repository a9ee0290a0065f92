#!/bin/bash
# Round-evidence call: parity suite, smoke, default bench line + launch list (gpu_check.sh), ncu --set full of the
# config-2 k_simulate launches and of k_estimate on config 4 (2M traces), configs 3-5 bench lines.
# usage: gpurun --timeout 3600 -- 'bash tools/gpu_round.sh <tag>'
tag=${1:-round}
bash tools/gpu_check.sh $tag
bash tools/gpu_ncu.sh 2 ${tag}_lane > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_lane.ncu-rep > gpurun_out/${tag}_lane_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/${tag}_lane.ncu-rep 60 > gpurun_out/${tag}_lane_lines.txt 2>&1
bash tools/gpu_est_prof.sh ${tag}_est_c4 > /dev/null 2>&1
for c in 3 4 5; do timeout 900 python bench.py --no-cpu --no-e2e --config $c > gpurun_out/bench_${tag}_c$c.json 2>/dev/null; cut -c1-300 gpurun_out/bench_${tag}_c$c.json; done
