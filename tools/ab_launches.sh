#!/bin/bash
# A/B of variants/<name>.so: ncu launch list of one garden frame each, then alternating bench runs.
mkdir -p gpurun_out
for lib in variants/*.so; do
  v=$(basename "$lib" .so)
  ADR_LIBRARY=$PWD/$lib timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/ab_$v.csv python tools/profile_frame.py --config ${CONFIG:-garden} > /dev/null 2>&1
  echo "== $v"; python tools/launches.py gpurun_out/ab_$v.csv | awk '{ if ($0 ~ /total/) print; else if ($(NF-7)+0 > 8) print }' | cut -c1-110
done
for r in $(seq ${REPS:-2}); do
  for lib in variants/*.so; do
    v=$(basename "$lib" .so)
    ADR_LIBRARY=$PWD/$lib timeout 300 python bench.py --config ${CONFIG:-garden} --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'fps', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
