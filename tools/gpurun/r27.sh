#!/bin/bash
# one-shot LL: parity + small-message sweep (2 GPUs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x -k "ll or repeated" > gpurun_out/r27_virtual.log 2>&1; echo "rc=$?" >> gpurun_out/r27_virtual.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "decompositions or bf16 or runtime_digests" > gpurun_out/r27_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r27_multi.log
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29541 tools/sweep.py --dtypes f32 --max-bytes 1048576 --iters 40 --out gpurun_out/r27_sweep2_auto.jsonl > gpurun_out/r27_sweep.log 2>&1
RBX_LL_ONESHOT_BYTES=0 $T --master-port 29542 tools/sweep.py --dtypes f32 --max-bytes 1048576 --iters 40 --mode ll --out gpurun_out/r27_sweep2_twoshot.jsonl >> gpurun_out/r27_sweep.log 2>&1
RBX_LL_ONESHOT_BYTES=65536 RBX_LL_AUTO_BYTES=1048576 $T --master-port 29543 tools/sweep.py --dtypes f32 --max-bytes 1048576 --iters 40 --out gpurun_out/r27_sweep2_os64.jsonl >> gpurun_out/r27_sweep.log 2>&1
