#!/bin/bash
# bf16x2 pack + dtype tile: parity, N=2 bench f32/bf16, bf16 sweep, N=1 bf16
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r33_virtual.log 2>&1; echo rc=$? >> gpurun_out/r33_virtual.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "bf16 or decompositions" > gpurun_out/r33_multi.log 2>&1; echo rc=$? >> gpurun_out/r33_multi.log
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for dt in f32 bf16; do
  $T --master-port 29581 bench.py --gpus 2 --steps 20 --warmup 5 --dtype $dt --no-nccl > gpurun_out/r33_bench2_$dt.log 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 --dtype bf16 --no-cpu-baseline > gpurun_out/r33_bench1_bf16.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 tools/sweep.py --dtypes bf16 --min-bytes 4194304 --iters 20 --out gpurun_out/r33_sweep2_bf16.jsonl > gpurun_out/r33_sweep.log 2>&1
