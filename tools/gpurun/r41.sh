#!/bin/bash
# stream ordering across launches: full GPU suites on 2 GPUs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r41_gpu.log 2>&1; echo rc=$? >> gpurun_out/r41_gpu.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 tools/hook_overhead.py > gpurun_out/r41_hook.log 2>&1
