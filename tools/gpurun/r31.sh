#!/bin/bash
# 2 GPUs: full parity suites (LL bf16 packing, local grid 1/SM), N=1 bench + ncu, bf16 small sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r31_virtual.log 2>&1; echo rc=$? >> gpurun_out/r31_virtual.log
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ddp.py -q > gpurun_out/r31_multi.log 2>&1; echo rc=$? >> gpurun_out/r31_multi.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r31_bench1.log 2>&1
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/r31_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r31_launches.csv $CMD > gpurun_out/r31_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rbx_local -s 4 -c 1 -o gpurun_out/r31_prof_local $CMD > gpurun_out/r31_ncu_full.log 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29561 tools/sweep.py --dtypes bf16,f32 --max-bytes 4194304 --iters 30 --out gpurun_out/r31_sweep2_small.jsonl > gpurun_out/r31_sweep.log 2>&1
