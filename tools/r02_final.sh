#!/bin/bash
# GPU box: final evidence — GPU tests, smoke(), bench lines of every config, the
# reference arm, and a 2-rank gloo run of the multi-rank bench path.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
NO_TESTS=1 CONFIGS="garden truck playroom stress config1" bash tools/r02_bench.sh final
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err
echo "ref rc=$?"; tail -c 300 gpurun_out/ref_final.json
ADR_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gloo2_final.json 2> gpurun_out/gloo2_final.err
echo "gloo2 rc=$?"; tail -c 300 gpurun_out/gloo2_final.json
