#!/bin/bash
# round-2: small-message tuning at N=2 -- LL words per thread, LL/FUSED crossover
cd "$(dirname "$0")/../.."
tr() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$((29200+RANDOM%90)) "$@"; }
for w in 1 2 4 8; do RBX_LL_WPT=$w tr tools/sweep.py --iters 20 --dtypes f32 --max-bytes 1048576 > gpurun_out/p_ll_wpt$w.jsonl 2>> gpurun_out/p.err; done
RBX_LL_AUTO_BYTES=0 tr tools/sweep.py --iters 20 --dtypes f32 --max-bytes 4194304 > gpurun_out/p_fused_small.jsonl 2>> gpurun_out/p.err
