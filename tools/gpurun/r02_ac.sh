#!/bin/bash
# round-2 (session 2): kernel launch + completion cost by kind of peer access (2 GPUs)
cd "$(dirname "$0")/../.."
(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o completion_probe completion_probe.cu)
timeout 300 ./tools/completion_probe > gpurun_out/ac_completion.jsonl 2> gpurun_out/ac.err
