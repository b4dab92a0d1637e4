#!/bin/bash
# 4 GPUs: full multi-GPU parity suite (incl. LL), fair sweeps at 2 and 4, buckets, bench N=2/4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/r29_multi.log 2>&1; echo rc=$? >> gpurun_out/r29_multi.log
for n in 2 4; do
timeout 300 $T --nproc-per-node $n --master-port 2961$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r29_bench$n.log 2>&1
timeout 1200 $T --nproc-per-node $n --master-port 2962$n tools/sweep.py --iters 20 --out gpurun_out/r29_sweep$n.jsonl > gpurun_out/r29_sweep$n.log 2>&1
timeout 300 $T --nproc-per-node $n --master-port 2963$n tools/buckets.py > gpurun_out/r29_buckets$n.log 2>&1
done
