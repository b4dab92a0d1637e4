#!/bin/bash
# 2 GPUs: is the host ahead of the device in bench.py's timed launches? spin 100k vs 1M cycles
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for rep in 1 2; do
for c in 100000 1000000; do
BENCH_SPIN_CYCLES=$c timeout 200 $T --master-port 2980$rep bench.py --gpus 2 --no-nccl --steps 30 > gpurun_out/r52_spin${c}_$rep.log 2>&1
done; done
