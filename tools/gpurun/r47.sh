#!/bin/bash
# 2 GPUs: prologue study (raw traces of both ranks)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2 --master-port 29741 tools/entry_study.py > gpurun_out/r47_entry.log 2>&1
