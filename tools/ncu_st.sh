#!/bin/bash
# ncu --set full of the supertile binning kernels of one garden frame.
tag=${1:-st}
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"k_st_|radix_downsweep" -o gpurun_out/ncu_${tag} -f python tools/profile_frame.py --config garden > gpurun_out/ncu_${tag}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_${tag}.log
