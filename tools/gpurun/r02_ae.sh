#!/bin/bash
# round-2 (session 2): N=1 e2e anatomy: host link one/both directions, copy-only and real window pipelines by lanes x windows x taper
cd "$(dirname "$0")/../.."
timeout 600 python tools/e2e_probe.py > gpurun_out/ae_e2e_probe.jsonl 2> gpurun_out/ae.err
timeout 600 python tools/e2e_probe.py --ranks 1 --n 25600000 --windows 4,8,16,32 > gpurun_out/ae_e2e_probe_1buf.jsonl 2>> gpurun_out/ae.err
