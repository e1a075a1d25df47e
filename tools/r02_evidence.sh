#!/bin/bash
# GPU box: evidence at the current code -> gpurun_out/ (launch lists per config,
# ncu --set full of one garden frame, compute-sanitizer runs).
mkdir -p gpurun_out
for c in ${CONFIGS:-garden truck playroom stress config1}; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_r02_$c.csv python tools/profile_frame.py --config $c > gpurun_out/prof_r02_$c.log 2>&1
  echo "launches $c rc=$?"
done
if [ -z "$NO_FULL" ]; then
timeout 1500 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o gpurun_out/full_r02 -f python tools/profile_frame.py --config garden > gpurun_out/full_r02.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/full_r02.log
fi
if [ -z "$NO_SAN" ]; then bash tools/sanitize.sh; fi
