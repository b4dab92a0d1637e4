#!/bin/bash
# 4 GPUs: reference in-process collective tests, multi-GPU parity, LL host cost, small sweeps N=2/4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_collectives_api.py -q > gpurun_out/r39_api.log 2>&1; echo rc=$? >> gpurun_out/r39_api.log
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ddp.py -q > gpurun_out/r39_multi.log 2>&1; echo rc=$? >> gpurun_out/r39_multi.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $T --nproc-per-node 2 --master-port 29641 tools/hook_overhead.py > gpurun_out/r39_hook.log 2>&1
for n in 2 4; do
timeout 600 $T --nproc-per-node $n --master-port 2965$n tools/sweep.py --dtypes f32,bf16 --max-bytes 4194304 --iters 30 --out gpurun_out/r39_sweep${n}_small.jsonl > gpurun_out/r39_sweep$n.log 2>&1
done
