#!/bin/bash
# GPU box: parity tests (first failure stops), then the ncu launch list of one garden frame and a short bench.
tag=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_${tag}.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/pytest_${tag}.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv python tools/profile_frame.py --config garden > gpurun_out/prof_${tag}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/prof_${tag}.log; python tools/launches.py gpurun_out/launches_${tag}.csv
if [ -z "$NO_BENCH" ]; then
timeout 600 python bench.py --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
echo "bench rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_${tag}.json').read().strip().splitlines()[-1]);print('fps',d['value'],'e2e',d.get('e2e',{}).get('value'),'clk',d['clocks'])"; tail -3 gpurun_out/bench_${tag}.err
fi
