#!/bin/bash
# round-2: N=1 local kernel cache policies, twice each (noise)
cd "$(dirname "$0")/../.."
for rep in 1 2; do for h in 0 3 4; do
  RBX_LOCAL_HINT=$h timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/q_bench1_h${h}_r$rep.json 2>> gpurun_out/q.err
done; done
