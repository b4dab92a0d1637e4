#!/bin/bash
# e2e (host buffers) pipeline depth: 8 / 16 / 32 windows at N=1 and N=2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 8 16 32; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-chunks $c > gpurun_out/r34_bench1_c$c.log 2>&1
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 2 --steps 10 --warmup 3 --no-nccl --e2e-chunks $c > gpurun_out/r34_bench2_c$c.log 2>&1
done
