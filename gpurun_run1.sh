nproc; lscpu | grep "Model name"
timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --traces 100000 2>&1 | tail -8
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -8 gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json
