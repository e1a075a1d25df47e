#!/bin/bash
# Functional test of bench.py's multi-rank path on a one-GPU box: two ranks on device 0 over gloo.
mkdir -p gpurun_out
for c in ${CONFIGS:-garden playroom}; do
ADR_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/gloo2_$c.json 2> gpurun_out/gloo2_$c.err
echo "gloo2 $c rc=$?"; tail -c 700 gpurun_out/gloo2_$c.json; tail -3 gpurun_out/gloo2_$c.err
done
