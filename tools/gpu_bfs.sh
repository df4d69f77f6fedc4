#!/bin/bash
# Quick GPU pass for search-kernel work: timings of the default search on C3
# objectives, the launch list of the same run (per-kernel device times), and
# the whole-space parity tests.  Outputs under gpurun_out/ with suffix $1.
set -u
S=${1:-x}
mkdir -p gpurun_out
timeout 300 python tools/time_bnb.py > gpurun_out/time_$S.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$S.csv \
  python tools/time_bnb.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullspace.py tests/test_gpu_parity.py -q -x ${PYTEST_ARGS:-} \
  > gpurun_out/test_$S.log 2>&1
tail -2 gpurun_out/test_$S.log
cat gpurun_out/time_$S.log | tail -3
