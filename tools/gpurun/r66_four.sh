#!/bin/bash
# 4 GPUs: bench.py --gpus 8 end to end with two ranks per GPU (functional check of the N=8 bench path)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29995 bench.py --gpus 8 --steps 5 --warmup 3 > gpurun_out/r66_bench8_shared.log 2>&1; echo rc=$? >> gpurun_out/r66_bench8_shared.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29996 bench.py --impl reference --gpus 8 --steps 3 --warmup 1 > gpurun_out/r66_ref8.log 2>&1; echo rc=$? >> gpurun_out/r66_ref8.log
