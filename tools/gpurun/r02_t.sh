#!/bin/bash
# round-2: the whole GPU suite on a 4-GPU box (per-process ranks on their own GPUs up to world 4: real NVLink)
cd "$(dirname "$0")/../.."
timeout 2700 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/t_pytest4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_pytest4.log
