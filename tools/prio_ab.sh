#!/bin/bash
for r in 1 2; do for p in none alt first; do
  ADR_STREAM_PRIO=$p timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p', 'fps', round(d['value'],1))"
done; done
for n in 3 5 6; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --streams $n 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('streams $n', 'fps', round(d['value'],1))"
done
