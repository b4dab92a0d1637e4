#!/bin/bash
# round-2 (session 2): the N=8 bench path with the final code on a 4-GPU box (two ranks per GPU): functional, not a measurement
cd "$(dirname "$0")/../.."
s=$(date +%s); timeout 1200 python bench.py --gpus 8 --steps 5 --warmup 3 > gpurun_out/aw_bench8_shared.json 2> gpurun_out/aw.err; echo "rc=$? wall=$(( $(date +%s)-s ))s" > gpurun_out/aw_wall.txt
