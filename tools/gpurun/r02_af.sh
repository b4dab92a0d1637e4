#!/bin/bash
# round-2 (session 2): N=1 e2e window pipeline: window-edge alignment x windows x taper (lanes 1)
cd "$(dirname "$0")/../.."
timeout 600 python tools/e2e_probe.py --windows 4,6,8,12,16,24 > gpurun_out/af_e2e_probe.jsonl 2> gpurun_out/af.err
timeout 600 python tools/e2e_probe.py --ranks 1 --n 25600000 --windows 4,8,12,16,32 > gpurun_out/af_e2e_probe_1buf.jsonl 2>> gpurun_out/af.err
