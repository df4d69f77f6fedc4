#!/bin/bash
# Full ncu capture of the frontier kernel (bfs_kernel) on the bench's headline
# instance; raw + SASS/CUDA-source CSVs and a summary under gpurun_out/
# (suffix $1).  LOOM_B200_LIB selects an experiment build; PROF_ARGS go to
# tools/prof_bnb.py.  Plain launches (LOOM_NO_GRAPH=1): ncu does not profile
# the cooperative kernel node of the search graph; the kernel is the same.
# The .ncu-rep is kept only with KEEP=1 (gpurun copies back at most 64 MiB).
set -u
S=${1:-x}
mkdir -p gpurun_out
LOOM_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfs_kernel -s 1 -c 1 \
  -o gpurun_out/fr_$S -f python tools/prof_bnb.py ${PROF_ARGS:-} > gpurun_out/ncu_fr_$S.log 2>&1
ncu -i gpurun_out/fr_$S.ncu-rep --page raw --csv > gpurun_out/fr_${S}_raw.csv 2>/dev/null
ncu -i gpurun_out/fr_$S.ncu-rep --page source --csv --print-source sass > gpurun_out/fr_${S}_sass.csv 2>/dev/null
ncu -i gpurun_out/fr_$S.ncu-rep --page source --csv --print-source cuda > gpurun_out/fr_${S}_cuda.csv 2>/dev/null
python tools/ncu_hot.py gpurun_out/fr_$S 40 > gpurun_out/fr_${S}_hot.txt 2>&1
gzip -f gpurun_out/fr_${S}_sass.csv
[ "${KEEP:-0}" = 1 ] || rm -f gpurun_out/fr_$S.ncu-rep
head -20 gpurun_out/fr_${S}_hot.txt
