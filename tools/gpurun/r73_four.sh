#!/bin/bash
# 4 GPUs: 16-byte loads in flight per thread, 8 (default) vs 12 (RBX_LD_DEPTH build variant), N=2/4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for rep in 1 2; do
timeout 200 $T --nproc-per-node $n --master-port 2998$n bench.py --gpus $n --no-nccl --curve 0 --steps 30 > gpurun_out/r73_b${n}_d8_$rep.log 2>&1
RBX_LIB_PATH=$PWD/paper_1708_02188_b200/librbx_d12.so timeout 200 $T --nproc-per-node $n --master-port 2998$n bench.py --gpus $n --no-nccl --curve 0 --steps 30 > gpurun_out/r73_b${n}_d12_$rep.log 2>&1
done; done
