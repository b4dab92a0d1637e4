#!/bin/bash
# round-2 (session 2): final code on a 4-GPU box: whole GPU suite (worlds 2/4/8 over NVLink), full bench lines N=2/N=4
cd "$(dirname "$0")/../.."
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/ap_pytest4.log 2>&1; echo rc=$? >> gpurun_out/ap_pytest4.log
timeout 900 python bench.py --gpus 2 > gpurun_out/ap_bench2.json 2> gpurun_out/ap_bench2.err
timeout 900 python bench.py --gpus 4 > gpurun_out/ap_bench4.json 2> gpurun_out/ap_bench4.err
