#!/bin/bash
# The driver's other invocations: reference arm, torchrun launch, another config.
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tail -1 | cut -c1-600
echo "ref rc=$?"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-300
echo "torchrun rc=$?"
timeout 400 python bench.py --config truck --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | cut -c1-400
echo "truck rc=$?"
