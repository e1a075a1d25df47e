#!/bin/bash
# Throughput A/B: bench.py (views in flight, no CPU baseline / e2e) for every
# variants/<name>.so, alternating, REPS rounds.  usage (under gpurun): bash tools/variant_bench.sh
for r in $(seq ${REPS:-2}); do
  for lib in variants/*.so; do
    v=$(basename "$lib" .so)
    ADR_LIBRARY=$PWD/$lib timeout 300 python bench.py --steps 120 --warmup 8 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'fps', round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
