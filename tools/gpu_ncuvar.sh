#!/bin/bash
# ncu --set full SASS source page of k_ff_lane (config 2) for every build/var/*.so (-> gpurun_out/var_<name>_src.csv)
cp paper_2508_18556_b200/libmig.so /tmp/libmig_orig.so
for v in build/var/*.so; do
  n=$(basename $v .so)
  cp $v paper_2508_18556_b200/libmig.so
  bash tools/gpu_ffncu.sh var_$n
done
cp /tmp/libmig_orig.so paper_2508_18556_b200/libmig.so
