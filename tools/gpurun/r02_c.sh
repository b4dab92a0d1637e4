#!/bin/bash
# round-2: fixed-cost anatomy on the device clock, carveout A/B
cd "$(dirname "$0")/../.."
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$1 tools/gap_probe.py; }
RBX_CARVEOUT=-1 run 29601 > gpurun_out/c_gap_default.jsonl 2> gpurun_out/c_gap.err
RBX_CARVEOUT=50 run 29602 > gpurun_out/c_gap_50.jsonl 2>> gpurun_out/c_gap.err
RBX_CARVEOUT=100 run 29603 > gpurun_out/c_gap_100.jsonl 2>> gpurun_out/c_gap.err
RBX_CARVEOUT=-1 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --curve 0 --no-cpu-baseline > gpurun_out/c_bench2_cdef.json 2> gpurun_out/c_bench.err
RBX_CARVEOUT=50 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --curve 0 --no-cpu-baseline > gpurun_out/c_bench2_c50.json 2>> gpurun_out/c_bench.err
