mkdir -p gpurun_out
export LOOM_STATS_READ=1
for v in st_default st_nobound; do
  export LOOM_B200_LIB=paper_2501_16634_b200/_build/variants/$v/libloom_b200.so
  echo "== $v"
  timeout 120 python tools/time_search.py --config c3 --reps 2
  timeout 120 python tools/time_search.py --config c3 --reps 2 --plans 68719476736
  timeout 120 python tools/time_search.py --config c3 --reps 2 --begin 500000000000 --plans 68719476736
done
