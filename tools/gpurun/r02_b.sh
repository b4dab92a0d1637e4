#!/bin/bash
# round-2: bench at N=4 (self-launch), fused-kernel latency trace at N=2
cd "$(dirname "$0")/../.."
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/b_bench4.json 2> gpurun_out/b_bench4.err; echo "rc=$?" >> gpurun_out/b_bench4.err
RBX_TRACE=1 LAT_MODES=fused,ll LAT_SIZES=1,262144,4194304,25600000 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 tools/latency_multi.py > gpurun_out/b_lat2.jsonl 2> gpurun_out/b_lat2.err
RBX_TRACE=1 LAT_MODES=fused LAT_SIZES=1,25600000 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29534 tools/latency_multi.py > gpurun_out/b_lat4.jsonl 2> gpurun_out/b_lat4.err
