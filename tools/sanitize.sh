#!/usr/bin/env bash
# compute-sanitizer over every kernel family on small problems (run under
# gpurun).  memcheck: out-of-bounds / misaligned accesses; racecheck and
# synccheck: shared-memory hazards and barrier misuse in the CTA-cooperative
# parts (warp DP, block reduction, Pareto guard staging).
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY: 0 errors' gpurun_out/sanitize_$tool.log) clean summaries; $(tail -1 gpurun_out/sanitize_$tool.log)"
done
