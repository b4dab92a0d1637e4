#!/bin/bash
# 2 GPUs: reference in-process collective tests with up to 2 ranks per GPU (worlds 2, 3, 4)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_collectives_api.py tests/test_gpu_multi.py -k "not bucket and not calib and not crash and not mismatch_abort" -q --durations=5 > gpurun_out/r69_api_2gpu.log 2>&1; echo rc=$? >> gpurun_out/r69_api_2gpu.log
