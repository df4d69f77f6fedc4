#!/bin/bash
# ncu --set full of the C4 batch kernel and the C5 Pareto kernels (the second
# call of each: tools/prof_c4c5.py), raw CSVs under gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"bnb_kernel" \
  -s 1 -c 1 -o gpurun_out/c4c5 -f python tools/prof_c4c5.py > gpurun_out/ncu_c4c5.log 2>&1
ncu -i gpurun_out/c4c5.ncu-rep --page raw --csv > gpurun_out/c4c5_raw.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c4c5_launches.csv python tools/prof_c4c5.py > /dev/null 2>&1
rm -f gpurun_out/c4c5.ncu-rep
tail -3 gpurun_out/ncu_c4c5.log
