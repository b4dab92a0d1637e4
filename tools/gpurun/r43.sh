#!/bin/bash
# 2 GPUs: copy-engine peer copy ceiling (one and both directions)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/ce_probe.py --mb 51.2 > gpurun_out/r43_ce_51.jsonl 2>&1
timeout 300 python tools/ce_probe.py --mb 204.8 --streams 1,4 > gpurun_out/r43_ce_204.jsonl 2>&1
