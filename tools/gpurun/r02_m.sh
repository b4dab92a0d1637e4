#!/bin/bash
# round-2: NVML NVLink data/raw counters in the real bidirectional run, final N=2/4 lines, randomised parity on 4 GPUs
cd "$(dirname "$0")/../.."
tr() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29500+RANDOM%90)) "$@"; }
tr 2 tools/nvlink_counters.py --iters 50 > gpurun_out/m_counters2.jsonl 2>> gpurun_out/m.err
tr 4 tools/nvlink_counters.py --iters 50 > gpurun_out/m_counters4.jsonl 2>> gpurun_out/m.err
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/m_bench2.json 2>> gpurun_out/m.err
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/m_bench4.json 2>> gpurun_out/m.err
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -k "randomised or fused_kernel" > gpurun_out/m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/m_pytest.log
