#!/bin/bash
# round-2 (session 2): reduce_scatter / allgather through the specialised kernel: parity (worlds 2/4) and RS/AG busbw at N=2/4
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_collectives_api.py -m gpu -q -x > gpurun_out/ai_pytest.log 2>&1; echo rc=$? >> gpurun_out/ai_pytest.log
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --curve 0 --no-nccl --no-cpu-baseline > gpurun_out/ai_bench2.json 2> gpurun_out/ai_bench2.err
timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 --curve 0 --no-nccl --no-cpu-baseline > gpurun_out/ai_bench4.json 2> gpurun_out/ai_bench4.err
