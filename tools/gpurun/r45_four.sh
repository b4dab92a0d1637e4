#!/bin/bash
# 4 GPUs: dynamic work tiles parity (virtual + multi) and A/B at N=2 and N=4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
RBX_DYN=1 RBX_TILE=2048 timeout 1200 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_multi.py -q -x > gpurun_out/r45_pytest_dyn.log 2>&1; echo rc=$? >> gpurun_out/r45_pytest_dyn.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for rep in 1 2; do
for cfg in "0 1024" "0 2048" "1 1024" "1 2048" "1 3072" "1 4096"; do
set -- $cfg
RBX_DYN=$1 RBX_TILE=$2 timeout 200 $T --nproc-per-node $n --master-port 2973$n bench.py --gpus $n --no-nccl --steps 30 > gpurun_out/r45_b${n}_dyn$1_t$2_$rep.log 2>&1
done; done; done
