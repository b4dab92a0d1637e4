#!/bin/bash
# round-2: interpreter parity after the spill fix, local-kernel cache hints (N=1), fused-kernel ncu harness
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_virtual.py -m gpu -q -x > gpurun_out/h_pytest_virtual.log 2>&1; echo "rc=$?" >> gpurun_out/h_pytest_virtual.log
for h in 0 1 2 3; do
  RBX_LOCAL_HINT=$h timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/h_bench1_hint$h.json 2>> gpurun_out/h.err
done
timeout 300 python tools/fused_ncu.py > gpurun_out/h_fused_harness.json 2>> gpurun_out/h.err && \
timeout 900 ncu --set full --section Nvlink --section Nvlink_Tables --clock-control none --import-source on -k regex:rbx_fused_kernel -c 2 -o gpurun_out/h_fused_full python tools/fused_ncu.py --iters 1 > gpurun_out/h_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/h_ncu.log
tools/nvlink_ceiling 4 256 1024 > gpurun_out/h_ceil4.jsonl 2>> gpurun_out/h.err
for v in ld16 ld4; do
  for n in 2 4; do
    RBX_LIB_PATH=$PWD/paper_1708_02188_b200/librbx_$v.so timeout 600 python bench.py --gpus $n --steps 20 --warmup 5 --curve 0 --no-cpu-baseline --no-nccl > gpurun_out/h_bench${n}_$v.json 2>> gpurun_out/h.err
  done
done
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 --curve 0 --no-cpu-baseline --no-nccl > gpurun_out/h_bench4_ld8.json 2>> gpurun_out/h.err
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "all_decompositions or full_size" > gpurun_out/h_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/h_pytest_multi.log
for g in 1 0; do
  RBX_RINGS_GPU_FENCE=$g timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 --curve 0 --no-cpu-baseline --no-nccl --mode ring_dims > gpurun_out/h_bench4_rings_gpufence$g.json 2>> gpurun_out/h.err
done
