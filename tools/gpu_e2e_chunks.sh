#!/bin/bash
# e2e (mig_simulate_host) ms/step at several host-pipeline chunk sizes (config 2)
for cj in 2097152 4194304 8388608 16777216; do
  echo -n "chunk_jobs=$cj: "
  MIG_HOST_CHUNK_JOBS=$cj timeout 300 python bench.py --no-cpu --steps 5 --e2e-steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['e2e']['ms_per_step'],2), round(d['ms_per_step'],3))"
done
