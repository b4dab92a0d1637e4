#!/bin/bash
# round-2 (session 2): LL kernel without the local-memory fold copy: whole GPU suite on the 2-GPU box's first GPU... (all ranks share), then the N=2 small-size sweep
cd "$(dirname "$0")/../.."
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ar_pytest1.log 2>&1; echo rc=$? >> gpurun_out/ar_pytest1.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29633 tools/sweep.py --max-bytes 4194304 --iters 30 --out gpurun_out/ar_sweep2.jsonl > /dev/null 2>> gpurun_out/ar.err
