#!/usr/bin/env bash
# Run under gpurun (one GPU).  Produces the raw evidence summarised into
# profiles/ by tools/summarize_ncu.py:
#   gpurun_out/launches.csv     every launch of the bench command, device time
#                               + DRAM bytes + instructions (cold, serialised)
#   gpurun_out/prof_full.ncu-rep  ncu --set full of the C3 search kernel
#   gpurun_out/prof_scores.ncu-rep  ncu --set full of the estimate-stream kernel
#   gpurun_out/bench.json       one normal bench line (never under ncu)
set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
  --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -c 1 \
  -o gpurun_out/prof_full -f python tools/prof_search.py --plans 1099511627776 --repeat 1 > gpurun_out/prof_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:estimate_range -c 1 \
  -o gpurun_out/prof_scores -f python tools/time_scores.py --log2 26 --reps 1 --host-log2 10 > gpurun_out/prof_scores.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
