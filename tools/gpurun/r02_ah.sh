#!/bin/bash
# round-2 (session 2): final state on a 4-GPU box: whole GPU suite (worlds 2/4 over NVLink), full bench lines N=2/N=4, reference arm N=4
cd "$(dirname "$0")/../.."
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/ah_pytest4.log 2>&1; echo rc=$? >> gpurun_out/ah_pytest4.log
s=$(date +%s); timeout 900 python bench.py --gpus 2 > gpurun_out/ah_bench2.json 2> gpurun_out/ah_bench2.err; echo "rc=$? wall=$(( $(date +%s)-s ))s" >> gpurun_out/ah_walls.txt
s=$(date +%s); timeout 900 python bench.py --gpus 4 > gpurun_out/ah_bench4.json 2> gpurun_out/ah_bench4.err; echo "rc=$? wall=$(( $(date +%s)-s ))s" >> gpurun_out/ah_walls.txt
s=$(date +%s); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29611 bench.py --impl reference --gpus 4 --steps 5 --warmup 3 > gpurun_out/ah_ref4.json 2> gpurun_out/ah_ref4.err; echo "ref rc=$? wall=$(( $(date +%s)-s ))s" >> gpurun_out/ah_walls.txt
