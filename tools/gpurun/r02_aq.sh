#!/bin/bash
# round-2 (session 2): launch latency by launch shape (grid, parameter bytes, registers, PDL)
cd "$(dirname "$0")/../.."
(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o launch_probe launch_probe.cu)
timeout 300 ./tools/launch_probe > gpurun_out/aq_launch.jsonl 2> gpurun_out/aq.err
