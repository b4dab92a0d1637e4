#!/bin/bash
# round-2 (session 2): final full bench lines N=2/N=4 with the final code (LL epoch change included)
cd "$(dirname "$0")/../.."
timeout 900 python bench.py --gpus 2 > gpurun_out/ay_bench2.json 2> gpurun_out/ay_bench2.err
timeout 900 python bench.py --gpus 4 > gpurun_out/ay_bench4.json 2> gpurun_out/ay_bench4.err
