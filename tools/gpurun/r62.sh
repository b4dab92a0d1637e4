#!/bin/bash
# 2 GPUs: bound writes in flight with fence.sys every K dynamic tiles (RBX_FENCE_EVERY) + entry study
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for rep in 1 2; do
for k in 0 1 2 4 8; do
RBX_FENCE_EVERY=$k timeout 200 $T --master-port 2998$k bench.py --gpus 2 --no-nccl --curve 0 --steps 30 > gpurun_out/r62_fence${k}_$rep.log 2>&1
done; done
RBX_FENCE_EVERY=2 timeout 300 $T --master-port 29989 tools/entry_study.py > gpurun_out/r62_entry_fence2.log 2>&1
