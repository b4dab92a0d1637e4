#!/bin/bash
# round-2 (session 2): reduce-scatter pass depth A/B (16 vs 8 loads per thread) at N=2/4; RS+AG parity
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "reduce_scatter_allgather_pair" > gpurun_out/aj_pytest.log 2>&1; echo rc=$? >> gpurun_out/aj_pytest.log
for rep in 1 2; do
for lib in librbx.so librbx_rs8.so; do
  for n in 2 4; do
    RBX_LIB_PATH=$PWD/paper_1708_02188_b200/$lib timeout 600 python bench.py --gpus $n --steps 20 --warmup 5 --curve 0 --no-nccl --no-cpu-baseline > gpurun_out/aj_bench${n}_${lib%.so}_$rep.json 2>> gpurun_out/aj.err
  done
done
done
