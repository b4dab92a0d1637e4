#!/bin/bash
# round-2 (session 2): config 3 sweep at N=2 with the final code (fp32 + bf16, 4 KB - 1 GiB)
cd "$(dirname "$0")/../.."
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29651 tools/sweep.py --iters 12 --out gpurun_out/az_sweep2.jsonl > /dev/null 2> gpurun_out/az.err
