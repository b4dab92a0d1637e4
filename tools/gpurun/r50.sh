#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dp.py tests/test_gpu_ddp.py -q -x > gpurun_out/r50_dp_test.log 2>&1; echo rc=$? >> gpurun_out/r50_dp_test.log
