timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo rc=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_simulate -s 3 -c 1 -o gpurun_out/r01_sim_c2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo rc=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_estimate -s 3 -c 1 -o gpurun_out/r01_est_c4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config 4 --traces 2000000 > /dev/null 2>&1; echo rc=$?
timeout 600 python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err; echo rc=$?; cat gpurun_out/r01_bench.json
