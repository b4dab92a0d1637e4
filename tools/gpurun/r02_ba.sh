#!/bin/bash
# round-2 (session 2): final code, the remaining GPU test files on a 2-GPU box (ranks on separate GPUs)
cd "$(dirname "$0")/../.."
timeout 1200 python -m pytest tests/test_gpu_collectives_api.py tests/test_gpu_dp.py tests/test_gpu_ddp.py tests/test_gpu_oversub.py -m gpu -q -x > gpurun_out/ba_pytest2.log 2>&1; echo rc=$? >> gpurun_out/ba_pytest2.log
