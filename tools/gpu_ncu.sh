#!/bin/bash
# ncu --set full capture of the k_simulate kernels of one bench step (config $1, default 2), plus per-line source.
# usage: gpurun --timeout 1800 -- 'bash tools/gpu_ncu.sh <config> <tag> [kernel-regex]'
cfg=${1:-2}; tag=${2:-ncu}; kre=${3:-regex:k_simulate}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k "$kre" -c 2 \
  -o gpurun_out/$tag -f python bench.py --no-cpu --no-e2e --no-dynamic --config $cfg --steps 1 --warmup 0 > gpurun_out/$tag.log 2>&1
tail -3 gpurun_out/$tag.log
ls -la gpurun_out/$tag.ncu-rep
