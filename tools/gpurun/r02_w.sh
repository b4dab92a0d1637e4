#!/bin/bash
# round-2: e2e with runtime.host_empty buffers at N=1 and N=2
cd "$(dirname "$0")/../.."
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/w_bench1.json 2> gpurun_out/w.err
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --curve 0 --no-nccl --no-cpu-baseline > gpurun_out/w_bench2.json 2>> gpurun_out/w.err
