#!/bin/bash
# round-2 (session 2): same-box A/B of reduce_scatter / allgather alone: specialised fused kernel vs the step interpreter (RBX_FUSED_KERNEL=0)
cd "$(dirname "$0")/../.."
for rep in 1 2; do
for k in 1 0; do
  for n in 2 4; do
    RBX_FUSED_KERNEL=$k timeout 600 python bench.py --gpus $n --steps 20 --warmup 5 --curve 0 --no-nccl --no-cpu-baseline > gpurun_out/ak_bench${n}_fk${k}_$rep.json 2>> gpurun_out/ak.err
  done
done
done
