#!/bin/bash
# round-2 (session 2): LL vs FUSED crossover at N=2 and N=4 (64 KB - 1 MB per rank)
cd "$(dirname "$0")/../.."
tr() { n=$1; shift; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((28800+RANDOM%90)) "$@"; }
tr 2 tools/tune_multi.py --elems 16384,65536,131072,262144 --ops allreduce --modes ll,fused --nblocks 148 --threads 512 --iters 40 > gpurun_out/ax_tune2.txt 2>> gpurun_out/ax.err
tr 4 tools/tune_multi.py --elems 16384,65536,131072,262144 --ops allreduce --modes ll,fused --nblocks 148 --threads 512 --iters 40 > gpurun_out/ax_tune4.txt 2>> gpurun_out/ax.err
