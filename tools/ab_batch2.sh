for r in 1 2; do
 for v in old new; do
  for extra in "" "--batch-views 1"; do
   ADR_LIBRARY=$PWD/variants/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $extra 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); bp=d.get('batch_preprocess') or {}; print('$v', '$extra', 'fps', round(d['value'],1), 'pre/view', round(bp.get('ms_per_view',0),4), d['stages_ms']['preprocess'], d['clocks']['sm_mhz'])"
  done
 done
done
ADR_LIBRARY=$PWD/variants/new.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --streams 8 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new streams8 fps', round(d['value'],1))"
for bv in 1 8; do for r in 1 2; do
ADR_LIBRARY=$PWD/variants/new.so timeout 300 python bench.py --config config1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --batch-views $bv 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config1 bv $bv fps', round(d['value'],1))"
done; done
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -2
