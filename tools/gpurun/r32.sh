#!/bin/bash
# N=2: work tile size x dtype (fold_body's U vectors per thread only fill when tile >= U*512)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for dt in f32 bf16; do
for tile in 1024 2048 4096; do
  RBX_TILE=$tile $T --master-port 29571 bench.py --gpus 2 --steps 20 --warmup 5 --dtype $dt --no-nccl > gpurun_out/r32_bench2_${dt}_t$tile.log 2>&1
done
done
