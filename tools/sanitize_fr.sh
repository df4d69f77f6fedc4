#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the
# frontier-search driver, plus memcheck with the fallbacks forced.  Logs in
# gpurun_out/sanitizer_r2/.
set -u
mkdir -p gpurun_out/sanitizer_r2
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_fr.py \
    > gpurun_out/sanitizer_r2/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_r2/summary.txt
done
LOOM_BFS_CAP=64 LOOM_BNB_BUDGET=4096 timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 \
  python tools/sanitize_fr.py > gpurun_out/sanitizer_r2/memcheck_fallbacks.log 2>&1
echo "memcheck (fallbacks forced) rc=$?" >> gpurun_out/sanitizer_r2/summary.txt
cat gpurun_out/sanitizer_r2/summary.txt
for f in gpurun_out/sanitizer_r2/*.log; do echo "== $f"; tail -3 $f; done
