#!/bin/bash
# GPU-box check: parity tests + one ncu launch list of the bench frame.
# usage (under gpurun): bash tools/gpu_check.sh <tag> [config]
tag=${1:-run}; cfg=${2:-garden}
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider 2>&1 | tail -5
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv python tools/profile_frame.py --config $cfg > /dev/null 2>&1
echo "ncu rc=$?"
