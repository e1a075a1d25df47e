#!/bin/bash
# Batched stage 1: GPU tests, then garden frames/s at 1 / 4 / 8 views per stage-1 launch.
# usage (under gpurun): bash tools/batch_check.sh <tag>
tag=${1:-b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider > gpurun_out/pytest_batch_${tag}.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_batch_${tag}.log
for bv in 1 4 8; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --batch-views $bv \
      > gpurun_out/bench_${tag}_bv${bv}.json 2> gpurun_out/bench_${tag}_bv${bv}.err
  echo "bv=$bv rc=$?"; python - "$tag" "$bv" <<'PY'
import json,sys
try:
    d=json.loads(open(f"gpurun_out/bench_{sys.argv[1]}_bv{sys.argv[2]}.json").read().splitlines()[-1])
    print(d["value"], d["config"].get("batch_views"), json.dumps(d.get("batch_preprocess")), d["stages_ms"])
except Exception as e: print("no line", e)
PY
done
