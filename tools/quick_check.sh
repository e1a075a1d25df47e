#!/bin/bash
# Quick GPU iteration: parity tests (optionally a -k filter) + the ncu launch list of one garden frame.
# usage (under gpurun): bash tools/quick_check.sh <tag> [pytest -k expr]
tag=${1:-q}; kexpr=${2:-}
mkdir -p gpurun_out
if [ -n "$kexpr" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$kexpr" > gpurun_out/pytest_${tag}.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${tag}.log 2>&1
fi
echo "pytest rc=$?"; tail -12 gpurun_out/pytest_${tag}.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv python tools/profile_frame.py --config garden > gpurun_out/prof_${tag}.log 2>&1
echo "ncu rc=$?"; python tools/launches.py gpurun_out/launches_${tag}.csv
