#!/bin/bash
# 2 GPUs: LL one-shot vs two-shot for small messages (per-rank LL kernel form)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 300 $T --master-port 29791 tools/sweep.py --dtypes f32 --max-bytes 1048576 --iters 30 --out gpurun_out/r51_twoshot.jsonl > gpurun_out/r51_twoshot.log 2>&1
RBX_LL_ONESHOT_BYTES=65536 timeout 300 $T --master-port 29792 tools/sweep.py --dtypes f32 --max-bytes 1048576 --iters 30 --out gpurun_out/r51_oneshot.jsonl > gpurun_out/r51_oneshot.log 2>&1
RBX_TRACE=1 LAT_SIZES=1,16384 LAT_MODES=ll timeout 300 $T --master-port 29793 tools/latency_multi.py > gpurun_out/r51_lat_twoshot.log 2>&1
RBX_LL_ONESHOT_BYTES=65536 RBX_TRACE=1 LAT_SIZES=1,16384 LAT_MODES=ll timeout 300 $T --master-port 29794 tools/latency_multi.py > gpurun_out/r51_lat_oneshot.log 2>&1
