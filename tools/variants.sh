#!/bin/bash
# A/B kernel variants on the GPU box: every variants/<name>.so is run through a
# parity subset and one ncu-timed garden frame.
# usage (under gpurun): bash tools/variants.sh [pytest -k expr]
kexpr=${1:-"parity and not stage"}
mkdir -p gpurun_out
for lib in variants/*.so; do
  v=$(basename "$lib" .so)
  export ADR_LIBRARY=$PWD/$lib
  timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$kexpr" > gpurun_out/pytest_var_${v}.log 2>&1
  echo "== $v pytest rc=$? $(tail -1 gpurun_out/pytest_var_${v}.log)"
  timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/launches_var_${v}.csv python tools/profile_frame.py --config garden \
      > gpurun_out/prof_var_${v}.log 2>&1
  python tools/launches.py gpurun_out/launches_var_${v}.csv | grep -E "k_render|k_preprocess|total"
done
