#!/bin/bash
# Quick frames/s of the given configs (no e2e / CPU legs).  usage: CONFIGS="garden stress" bash tools/quick_bench.sh [bench args]
for c in ${CONFIGS:-garden}; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2> gpurun_out/qb_$c.err | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); bp=d.get('batch_preprocess') or {}; print('$c', 'fps', round(d['value'],1), 'render-only', round(d['render_only_value'],1), 'pre/view', round(bp.get('ms_per_view',0),4), d['clocks'])" || tail -3 gpurun_out/qb_$c.err
done
