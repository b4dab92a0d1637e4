#!/bin/bash
# LL argument cache: parity (1 + 2 GPUs), hook host cost, small-message sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r38_virtual.log 2>&1; echo rc=$? >> gpurun_out/r38_virtual.log
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ddp.py -q > gpurun_out/r38_multi.log 2>&1; echo rc=$? >> gpurun_out/r38_multi.log
T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29631 tools/hook_overhead.py > gpurun_out/r38_hook.log 2>&1
$T --master-port 29632 tools/sweep.py --dtypes f32,bf16 --max-bytes 1048576 --iters 30 --out gpurun_out/r38_sweep2_small.jsonl > gpurun_out/r38_sweep.log 2>&1
