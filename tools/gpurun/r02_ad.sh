#!/bin/bash
# round-2 (session 2): completion cost by number of CTAs touching the peer; LL one-shot vs two-shot at N=2
cd "$(dirname "$0")/../.."
(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o completion_probe completion_probe.cu)
timeout 300 ./tools/completion_probe > gpurun_out/ad_completion.jsonl 2> gpurun_out/ad.err
tr() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$((28800+RANDOM%90)) "$@"; }
tr tools/sweep.py --max-bytes 4194304 --dtypes f32 --iters 30 --out gpurun_out/ad_sweep_twoshot.jsonl > /dev/null 2>> gpurun_out/ad.err
RBX_LL_ONESHOT_BYTES=65536 tr tools/sweep.py --max-bytes 262144 --dtypes f32 --iters 30 --out gpurun_out/ad_sweep_oneshot.jsonl > /dev/null 2>> gpurun_out/ad.err
