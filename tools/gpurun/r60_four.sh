#!/bin/bash
# 4 GPUs: finer tail tiles (RBX_TAIL_SPLIT) parity + A/B at N=2/N=4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
RBX_TAIL_SPLIT=4 timeout 900 python -m pytest tests/test_gpu_virtual.py -k "full_size or graph" -q > gpurun_out/r60_pytest.log 2>&1; echo rc=$? >> gpurun_out/r60_pytest.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for rep in 1 2; do
for sp in 1 2 4 8; do
RBX_TAIL_SPLIT=$sp timeout 200 $T --nproc-per-node $n --master-port 2997$n bench.py --gpus $n --no-nccl --curve 0 --steps 30 > gpurun_out/r60_b${n}_split${sp}_$rep.log 2>&1
done; done; done
