#!/bin/bash
# Round-evidence call: parity suite, smoke, default bench line + launch list (gpu_check.sh); ncu --set full of the
# config-2 k_simulate launches (with source) and of k_estimate at full size on configs 3, 4 and 5 (the dominant
# kernel there); configs 3-5 bench lines; a 2-rank functional run of the multi-rank path (gloo, one shared GPU).
# usage: gpurun --timeout 3600 -- 'bash tools/gpu_round.sh <tag>'
tag=${1:-round}
bash tools/gpu_check.sh $tag
bash tools/gpu_ncu.sh 2 ${tag}_lane > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_lane.ncu-rep > gpurun_out/${tag}_lane_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/${tag}_lane.ncu-rep 60 > gpurun_out/${tag}_lane_lines.txt 2>&1
python tools/ncu_to_json.py gpurun_out/${tag}_lane.ncu-rep sim_ff='k_simulate_lane<3' sim_baseline='k_simulate_lane<0' \
  --source "profiles/${tag}_ncu_lane_c2.txt (ncu --set full --clock-control none, config 2, 1M traces, k_simulate_lane<FUSION_FISSION> and <BASELINE>, serialised by ncu)" > gpurun_out/ncu_config2.json
for c in 3 4 5; do
  timeout 900 ncu --set full --clock-control none -k regex:k_estimate -c 1 -o gpurun_out/${tag}_est_c$c -f \
    python bench.py --no-cpu --no-e2e --config $c --steps 1 --warmup 0 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_est_c$c.ncu-rep > gpurun_out/${tag}_est_c${c}_summary.txt 2>&1
  python tools/ncu_to_json.py gpurun_out/${tag}_est_c$c.ncu-rep k_estimate='k_estimate' \
    --source "profiles/${tag}_ncu_est_c$c.txt (ncu --set full --clock-control none, config $c at full size, k_estimate)" > gpurun_out/ncu_config$c.json
done
for c in 3 4 5; do timeout 900 python bench.py --no-cpu --no-e2e --config $c > gpurun_out/bench_${tag}_c$c.json 2>/dev/null; cut -c1-300 gpurun_out/bench_${tag}_c$c.json; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --dist-backend gloo > gpurun_out/bench_${tag}_2rank_gloo.json 2>/dev/null
cut -c1-200 gpurun_out/bench_${tag}_2rank_gloo.json
