#!/bin/bash
# 4 GPUs: bench N=2/4 with reduce-scatter / all-gather fields
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
timeout 400 $T --nproc-per-node $n --master-port 2996$n bench.py --gpus $n > gpurun_out/r68_bench$n.log 2>&1
done
