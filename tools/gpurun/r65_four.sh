#!/bin/bash
# 4 GPUs: the world-8 multi-GPU tests with two rank processes per GPU
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -k "decompositions or runtime_digests or full_size" -q --durations=10 > gpurun_out/r65_multi8.log 2>&1; echo rc=$? >> gpurun_out/r65_multi8.log
