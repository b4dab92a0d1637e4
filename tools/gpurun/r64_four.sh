#!/bin/bash
# 4 GPUs: bf16 bench lines (fp32 accumulation, one RNE) at N=2/4, with curves
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
timeout 300 $T --nproc-per-node $n --master-port 2999$n bench.py --gpus $n --dtype bf16 > gpurun_out/r64_bench${n}_bf16.log 2>&1
done
timeout 300 python bench.py --dtype bf16 --no-cpu-baseline > gpurun_out/r64_bench1_bf16.log 2>&1
