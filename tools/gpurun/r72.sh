#!/bin/bash
# 1 GPU: compute-sanitizer memcheck / racecheck / synccheck / initcheck over every kernel mode (virtual ranks)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
timeout -s KILL 500 $CS --tool $tool --error-exitcode 9 python tests/sanitize_workload.py > gpurun_out/r72_$tool.log 2>&1; echo rc=$? >> gpurun_out/r72_$tool.log
done
