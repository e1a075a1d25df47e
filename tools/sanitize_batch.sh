#!/bin/bash
# compute-sanitizer over tools/sanitize_frame.py (small frames incl. the batched path) and a
# 300K-Gaussian frame (multi-block look-back, batched stage 1 of two views).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_frame.py \
    > gpurun_out/sanbatch_${tool}.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanbatch_${tool}.log
done
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_frame.py 300000 \
    > gpurun_out/sanbatch_${tool}_300k.log 2>&1
  echo "$tool 300k rc=$?"; tail -2 gpurun_out/sanbatch_${tool}_300k.log
done
