#!/bin/bash
# 4 GPUs: CTA shape of the step kernel with dynamic tiles (148x512 vs 296x256 vs 148x256), N=2/4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
timeout 400 $T --nproc-per-node $n --master-port 2997$n tools/tune_multi.py --modes fused --nblocks 148,296 --threads 256,512 --elems 4194304,25600000 > gpurun_out/r70_tune$n.log 2>&1
done
