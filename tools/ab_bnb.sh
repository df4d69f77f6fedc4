for v in default tpw16 tpw256; do
  if [ $v != default ]; then export LOOM_B200_LIB=paper_2501_16634_b200/_build/variants/$v/libloom_b200.so; else unset LOOM_B200_LIB; fi
  timeout 300 python tools/time_bnb.py
done
