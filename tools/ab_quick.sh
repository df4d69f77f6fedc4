# Quick A/B of experiment builds on the C3 full space: bash tools/ab_quick.sh default u4 ...
for v in "$@"; do
  if [ $v != default ]; then export LOOM_B200_LIB=paper_2501_16634_b200/_build/variants/$v/libloom_b200.so; else unset LOOM_B200_LIB; fi
  timeout 120 python tools/time_search.py --config c3 --reps 5
done
