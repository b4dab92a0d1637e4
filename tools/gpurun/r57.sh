#!/bin/bash
# 1 GPU: 8 rank processes on one GPU (test_gpu_oversub) + smoke
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_oversub.py -q -x > gpurun_out/r57_oversub_1gpu.log 2>&1; echo rc=$? >> gpurun_out/r57_oversub_1gpu.log
nvidia-smi > gpurun_out/r57_smi_after.txt 2>&1
