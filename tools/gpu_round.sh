#!/bin/bash
# One GPU-box pass: GPU tests, the bench, the bench's launch list, and a full
# ncu capture of the branch-and-bound kernel.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/gputest.log 2>&1
  tail -3 gpurun_out/gputest.log
fi
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
LOOM_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs \
  > gpurun_out/bench_ncu.log 2>&1
K=${KERNEL:-bfs_kernel}
LOOM_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s 1 -c 1 \
  -o gpurun_out/${K}_full -f python tools/prof_bnb.py > gpurun_out/ncu_$K.log 2>&1
mv -f gpurun_out/${K}_full.ncu-rep gpurun_out/${K}_full.ncu-rep 2>/dev/null
ncu -i gpurun_out/${K}_full.ncu-rep --page raw --csv > gpurun_out/${K}_raw.csv 2>/dev/null
ncu -i gpurun_out/${K}_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${K}_sass.csv 2>/dev/null
cp gpurun_out/${K}_sass.csv gpurun_out/${K}_sass.csv.tmp; mv gpurun_out/${K}_sass.csv.tmp gpurun_out/${K}_sass.csv; python tools/ncu_hot.py gpurun_out/${K} 40 > gpurun_out/${K}_hot.txt 2>&1
gzip -f gpurun_out/${K}_sass.csv
[ "${KEEP:-0}" = 1 ] || rm -f gpurun_out/${K}_full.ncu-rep
ls -la gpurun_out
