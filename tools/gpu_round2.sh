#!/bin/bash
# Round-2 evidence in one call: GPU parity suite, smoke, ncu --set full of the config-2 lane kernels (k_ff_lane,
# k_base_lane) and of k_estimate at full size on configs 3-5 (-> gpurun_out/ncu_config*.json, copied into profiles/
# before the bench lines so their roofline.traffic is this build's), the default bench line, the ncu launch list of
# the config-2 step, configs 3/4/5 bench lines, a 2-rank functional run (gloo, one shared GPU).
# usage: gpurun --timeout 3600 -- 'bash tools/gpu_round2.sh <tag>'
tag=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tail -1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/${tag}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ff_lane|k_base_lane" -c 2 \
  -o gpurun_out/${tag}_lane -f python bench.py --no-cpu --no-e2e --no-dynamic --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_lane.ncu-rep > gpurun_out/${tag}_ncu_lane_c2.txt 2>&1
python tools/ncu_to_json.py gpurun_out/${tag}_lane.ncu-rep sim_ff='k_ff_lane' sim_baseline='k_base_lane' \
  --source "profiles/${tag}_ncu_lane_c2.txt (ncu --set full --clock-control none, config 2, 1M traces, k_ff_lane and k_base_lane, serialised by ncu)" > gpurun_out/ncu_config2.json
for c in 3 4 5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_estimate -c 1 -o gpurun_out/${tag}_est_c$c -f \
    python bench.py --no-cpu --no-e2e --config $c --steps 1 --warmup 0 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_est_c$c.ncu-rep > gpurun_out/${tag}_ncu_est_c$c.txt 2>&1
  python tools/ncu_to_json.py gpurun_out/${tag}_est_c$c.ncu-rep k_estimate='k_estimate' \
    --source "profiles/${tag}_ncu_est_c$c.txt (ncu --set full --clock-control none, config $c, k_estimate)" > gpurun_out/ncu_config$c.json
done
cp gpurun_out/ncu_config*.json profiles/
timeout 600 python bench.py > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err; tail -4 gpurun_out/${tag}_bench_c2.err
cut -c1-400 gpurun_out/${tag}_bench_c2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --no-cpu --no-e2e --no-dynamic --steps 3 --warmup 3 > /dev/null 2>&1
for c in 3 4 5; do
  timeout 900 python bench.py --no-e2e --config $c --steps 5 > gpurun_out/${tag}_bench_c$c.json 2>/dev/null
  cut -c1-300 gpurun_out/${tag}_bench_c$c.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --cpu-seconds 5 --cpu-seconds-dynamic 3 --e2e-steps 2 \
  > gpurun_out/${tag}_bench_c2_2ranks_sharedgpu_gloo.json 2> gpurun_out/${tag}_2rank.err
cut -c1-300 gpurun_out/${tag}_bench_c2_2ranks_sharedgpu_gloo.json; tail -3 gpurun_out/${tag}_2rank.err
