#!/bin/bash
# round-2: tapered host-pipeline windows (e2e) at N=1 and N=2
cd "$(dirname "$0")/../.."
for w in 8 16; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-chunks $w > gpurun_out/u_bench1_w$w.json 2>> gpurun_out/u.err; done
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --curve 0 --no-nccl --no-cpu-baseline > gpurun_out/u_bench2.json 2>> gpurun_out/u.err
