#!/bin/bash
# ncu --set full of config 4's lane launches (k_ff_lane FF+ER and FF, k_base_lane) with SASS source pages.
tag=${1:-c4lane}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_ff_lane|k_base_lane" -c 3 \
  -o gpurun_out/$tag -f python bench.py --no-cpu --no-e2e --no-dynamic --config 4 --steps 1 --warmup 0 > gpurun_out/$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/$tag.ncu-rep > gpurun_out/${tag}_summary.txt 2>&1
grep -E "==|duration|inst_issued|inst_executed.sum|per_inst|dram__bytes" gpurun_out/${tag}_summary.txt
for i in 0 1 2; do
  ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source=sass --launch-skip $i --launch-count 1 > gpurun_out/${tag}_src$i.csv 2>/dev/null
done
rm -f gpurun_out/$tag.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_estimate -c 1 -o gpurun_out/${tag}_est -f \
  python bench.py --no-cpu --no-e2e --config 4 --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_est.ncu-rep | grep -E "duration|inst_issued|inst_executed.sum|per_inst|dram__bytes"
ncu -i gpurun_out/${tag}_est.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_est_src.csv 2>/dev/null
rm -f gpurun_out/${tag}_est.ncu-rep
