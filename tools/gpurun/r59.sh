#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_virtual.py -k "graph or repeated" -q > gpurun_out/r59_graph.log 2>&1; echo rc=$? >> gpurun_out/r59_graph.log
