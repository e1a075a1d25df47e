#!/bin/bash
# GPU-box round check: parity tests, smoke, a bench line, the ncu launch list.
# usage (under gpurun): bash tools/round_check.sh <tag>
tag=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${tag}.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_${tag}.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_${tag}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1
echo "smoke rc=$?"; tail -3 gpurun_out/smoke_${tag}.log
timeout 600 python bench.py --steps 60 --warmup 5 > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_${tag}.json; tail -5 gpurun_out/bench_${tag}.err
timeout 400 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv python tools/profile_frame.py --config garden > gpurun_out/prof_${tag}.log 2>&1
echo "ncu rc=$?"; python tools/launches.py gpurun_out/launches_${tag}.csv
