#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c5.csv python bench.py --no-cpu --no-e2e --config 5 --steps 2 --warmup 3 > /dev/null 2>&1
echo "c5 launches: $(wc -l < gpurun_out/launches_c5.csv)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_estimate -c 1 -o gpurun_out/est_c4 -f python bench.py --no-cpu --no-e2e --config 4 --steps 1 --warmup 0 --traces 2000000 > gpurun_out/est_c4.log 2>&1
tail -2 gpurun_out/est_c4.log
