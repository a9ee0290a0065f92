timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --traces 300000 > gpurun_out/multi2.json 2> gpurun_out/multi2.err; echo rc=$?; tail -3 gpurun_out/multi2.err; cat gpurun_out/multi2.json | cut -c1-600
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_simulate -s 3 -c 1 -o gpurun_out/r01b_sim_c2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo rc=$?
