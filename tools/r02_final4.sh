#!/bin/bash
# GPU box: evidence at the batched-stage-1 code -> gpurun_out/ (GPU tests, smoke,
# bench lines of every config, reference arm, 2-rank gloo run, launch lists of one
# batched garden step and one single frame, ncu --set full of the batched step).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_f4.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_f4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_f4.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/smoke_f4.log
NO_TESTS=1 CONFIGS="garden truck playroom stress config1" bash tools/r02_bench.sh f4
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref_f4.json 2> gpurun_out/ref_f4.err
echo "ref rc=$?"; tail -c 300 gpurun_out/ref_f4.json
ADR_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gloo2_f4.json 2> gpurun_out/gloo2_f4.err
echo "gloo2 rc=$?"; tail -c 300 gpurun_out/gloo2_f4.json
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv \
  --log-file gpurun_out/launches_f4_garden_batch8.csv python tools/profile_frame.py --config garden --batch 8 > gpurun_out/prof_f4_b.log 2>&1
echo "launches batch rc=$?"
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv \
  --log-file gpurun_out/launches_f4_garden.csv python tools/profile_frame.py --config garden > gpurun_out/prof_f4_s.log 2>&1
echo "launches single rc=$?"
timeout 1500 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -c 14 -o gpurun_out/full_f4 -f python tools/profile_frame.py --config garden --batch 8 > gpurun_out/full_f4.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/full_f4.log
