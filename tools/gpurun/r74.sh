#!/bin/bash
# 1 GPU: ncu launch list (gpu__time_duration.sum, --clock-control none) of the N=1 bench, after a clean run
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r74_bench1.log 2>&1; echo rc=$? >> gpurun_out/r74_bench1.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r74_launches_n1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r74_ncu.log 2>&1; echo rc=$? >> gpurun_out/r74_ncu.log
