#!/bin/bash
# round-2 check: fused kernel parity on 2 GPUs, bench --gpus 2 (self-launch), fused vs generic A/B
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "fused or all_decompositions or bucket or bf16" > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/a_bench2.json 2> gpurun_out/a_bench2.err; echo "bench rc=$?" >> gpurun_out/a_bench2.err
RBX_FUSED_KERNEL=0 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --curve 0 --no-cpu-baseline > gpurun_out/a_bench2_generic.json 2> gpurun_out/a_bench2_generic.err
RBX_PDL=0 timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --curve 0 --no-cpu-baseline > gpurun_out/a_bench2_nopdl.json 2> gpurun_out/a_bench2_nopdl.err
