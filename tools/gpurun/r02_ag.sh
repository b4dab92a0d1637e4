#!/bin/bash
# round-2 (session 2): host pipeline with equal 64 KB-aligned windows: host-buffer parity tests, bench N=1 e2e
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_collectives_api.py tests/test_gpu_virtual.py -m gpu -q -x -k "host" > gpurun_out/ag_pytest.log 2>&1; echo rc=$? >> gpurun_out/ag_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ag_bench1.json 2> gpurun_out/ag.err
