#!/bin/bash
# Same-box A/B of variants/<name>.so on bench frames/s (alternating runs).
# usage (under gpurun): REPS=2 CONFIG=garden bash tools/ab_bench.sh [extra bench args]
mkdir -p gpurun_out
for r in $(seq ${REPS:-2}); do
  for lib in variants/*.so; do
    v=$(basename "$lib" .so)
    ADR_LIBRARY=$PWD/$lib timeout 300 python bench.py --config ${CONFIG:-garden} --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); bp=d.get('batch_preprocess') or {}; print('$v', 'fps', round(d['value'],1), 'pre/view ms', round(bp.get('ms_per_view',0),4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
