#!/bin/bash
# round-2 (session 2): N=1 e2e anatomy: host link one/both directions, 1 vs 2 streams, copy-only window pipeline, e2e
cd "$(dirname "$0")/../.."
timeout 600 python tools/e2e_probe.py > gpurun_out/ae_e2e_probe.jsonl 2> gpurun_out/ae.err
