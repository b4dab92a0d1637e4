#!/bin/bash
# 4 GPUs: the 8-rank per-process path with two ranks per GPU (time-sliced contexts)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 240 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 8 --master-port 29961 tests/oversub8.py > gpurun_out/r56_oversub8.log 2>&1; echo rc=$? >> gpurun_out/r56_oversub8.log
nvidia-smi > gpurun_out/r56_smi_after.txt 2>&1
