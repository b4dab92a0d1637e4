#!/bin/bash
# round-2 (session 2): which NCCL algorithm wins small allreduces at N=2, and NCCL without NVLS / per algorithm
cd "$(dirname "$0")/../.."
tr() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$((28800+RANDOM%90)) "$@"; }
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING tr tools/sweep.py --max-bytes 65536 --dtypes f32 --iters 30 --out gpurun_out/as_default.jsonl > gpurun_out/as_default.log 2>&1
NCCL_NVLS_ENABLE=0 tr tools/sweep.py --max-bytes 65536 --dtypes f32 --iters 30 --out gpurun_out/as_nonvls.jsonl > /dev/null 2>> gpurun_out/as.err
NCCL_ALGO=Ring tr tools/sweep.py --max-bytes 65536 --dtypes f32 --iters 30 --out gpurun_out/as_ring.jsonl > /dev/null 2>> gpurun_out/as.err
NCCL_ALGO=Tree tr tools/sweep.py --max-bytes 65536 --dtypes f32 --iters 30 --out gpurun_out/as_tree.jsonl > /dev/null 2>> gpurun_out/as.err
