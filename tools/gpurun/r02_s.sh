#!/bin/bash
# round-2: N=1 host-buffer pipeline windows
cd "$(dirname "$0")/../.."
for w in 4 8 16 32; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-chunks $w > gpurun_out/s_bench1_w$w.json 2>> gpurun_out/s.err
done
