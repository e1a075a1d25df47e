#!/bin/bash
# compute-sanitizer over tools/sanitize_frame.py (one tool per run).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_frame.py \
    > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_${tool}.log
done
