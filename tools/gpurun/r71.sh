#!/bin/bash
# 1 GPU: the whole GPU suite as the round-end driver runs it on a single B200, plus smoke
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r71_gpu_1gpu.log 2>&1; echo rc=$? >> gpurun_out/r71_gpu_1gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r71_smoke.log 2>&1; echo rc=$? >> gpurun_out/r71_smoke.log
