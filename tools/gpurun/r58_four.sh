#!/bin/bash
# 4 GPUs: NCCL comparison column with NVLS forced on / off (ours unchanged), 1 MB..1 GiB fp32
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
NCCL_NVLS_ENABLE=1 NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 600 $T --master-port 29971 tools/sweep.py --dtypes f32 --min-bytes 1048576 --iters 20 --out gpurun_out/r58_nvls1.jsonl > gpurun_out/r58_nvls1.log 2>&1
NCCL_NVLS_ENABLE=0 timeout 600 $T --master-port 29972 tools/sweep.py --dtypes f32 --min-bytes 1048576 --iters 20 --out gpurun_out/r58_nvls0.jsonl > gpurun_out/r58_nvls0.log 2>&1
