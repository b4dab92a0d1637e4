#!/bin/bash
# 2 GPUs: dynamic work tiles (RBX_DYN) parity + A/B at N=2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
RBX_DYN=1 timeout 900 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_multi.py -q -x > gpurun_out/r44_pytest_dyn.log 2>&1; echo rc=$? >> gpurun_out/r44_pytest_dyn.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for rep in 1 2 3; do
for d in 0 1; do
RBX_DYN=$d timeout 200 $T --master-port 2971$rep bench.py --gpus 2 --no-nccl --steps 30 > gpurun_out/r44_b2_dyn${d}_$rep.log 2>&1
done; done
for tile in 512 2048 4096; do
RBX_DYN=1 RBX_TILE=$tile timeout 200 $T --master-port 29720 bench.py --gpus 2 --no-nccl --steps 30 > gpurun_out/r44_b2_dyn1_tile$tile.log 2>&1
done
