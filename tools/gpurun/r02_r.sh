#!/bin/bash
# round-2: LL words per thread at N=4 (small messages), then the N=2 small-size sweep with the new default
cd "$(dirname "$0")/../.."
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29100+RANDOM%90)) "$@"; }
for w in 2 4; do RBX_LL_WPT=$w tr 4 tools/sweep.py --iters 20 --dtypes f32,bf16 --max-bytes 1048576 > gpurun_out/r_ll4_wpt$w.jsonl 2>> gpurun_out/r.err; done
tr 2 tools/sweep.py --iters 20 --dtypes bf16 --max-bytes 1048576 > gpurun_out/r_ll2_bf16_wpt2.jsonl 2>> gpurun_out/r.err
