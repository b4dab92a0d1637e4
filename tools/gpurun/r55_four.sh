#!/bin/bash
# 4 GPUs: per-step pass tiles -- parity (virtual + multi) and every mode at N=2/N=4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_multi.py -q -x > gpurun_out/r55_pytest.log 2>&1; echo rc=$? >> gpurun_out/r55_pytest.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for m in fused ring_dims fused_pull push; do
timeout 200 $T --nproc-per-node $n --master-port 2995$n bench.py --gpus $n --mode $m --no-nccl --curve 0 > gpurun_out/r55_b${n}_$m.log 2>&1
done; done
