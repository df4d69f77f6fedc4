# A/B timing of experiment builds (python -m paper_2501_16634_b200.build --variant NAME -D...):
#   bash tools/ab_search.sh [variant ...]    ("default" = the in-tree library)
mkdir -p gpurun_out
for v in ${@:-default}; do
  if [ $v != default ]; then export LOOM_B200_LIB=paper_2501_16634_b200/_build/variants/$v/libloom_b200.so; else unset LOOM_B200_LIB; fi
  echo "== $v"
  timeout 120 python tools/time_search.py --config c3 --reps 5
  timeout 120 python tools/time_search.py --config c3 --reps 3 --plans 68719476736
  timeout 120 python tools/time_search.py --config c3 --reps 3 --begin 500000000000 --plans 68719476736
  timeout 120 python tools/time_search.py --config c5 --reps 5 --objective '{"constraint": "MIN_COST"}'
  timeout 200 python tools/time_c4.py 2>&1 | tail -1
done
