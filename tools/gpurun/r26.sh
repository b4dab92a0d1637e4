#!/bin/bash
# LL mode: parity (1 GPU virtual + 2-GPU multi), latency timeline, launch-cost probe, sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 ./tools/entry_probe > gpurun_out/r26_entry.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x -k "ll or repeated or decompositions" > gpurun_out/r26_virtual.log 2>&1; echo "rc=$?" >> gpurun_out/r26_virtual.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "decompositions or bf16 or runtime_digests" > gpurun_out/r26_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r26_multi.log
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
RBX_TRACE=1 $T --master-port 29531 tools/latency_multi.py > gpurun_out/r26_latency.log 2>&1
$T --master-port 29532 tools/sweep.py --dtypes f32,bf16 --max-bytes 67108864 --out gpurun_out/r26_sweep2_auto.jsonl > gpurun_out/r26_sweep.log 2>&1
$T --master-port 29533 tools/sweep.py --dtypes f32 --max-bytes 1048576 --mode ll --out gpurun_out/r26_sweep2_ll.jsonl >> gpurun_out/r26_sweep.log 2>&1
