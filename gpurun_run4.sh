timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_simulate -s 3 -c 1 -o gpurun_out/prof_sim_c2_v2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full2.log 2>&1; echo rc=$?
timeout 300 python bench.py --no-cpu --no-e2e --config 4 2>&1 | tail -1
timeout 300 python bench.py --no-cpu --no-e2e --config 3 2>&1 | tail -1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_estimate -s 3 -c 1 -o gpurun_out/prof_est_c4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config 4 --traces 2000000 > gpurun_out/ncu_full3.log 2>&1; echo rc=$?
