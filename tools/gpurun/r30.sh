#!/bin/bash
# N=1 local kernel: CTAs per SM (1 vs occupancy 2), 3 repeats each
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2 3; do
for c in 1 0; do
  RBX_LOCAL_CTAS_PER_SM=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r30_bench1_cps$c.$rep.log 2>&1
done
done
