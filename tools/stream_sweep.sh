#!/bin/bash
# bench.py at 1..4 (or $STREAMS) views in flight (no CPU baseline / e2e): frames/s per setting
for k in ${STREAMS:-1 2 3 4}; do
  timeout 300 python bench.py --steps 80 --warmup 8 --streams $k --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('streams', $k, 'fps', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), d['clocks'])"
done
