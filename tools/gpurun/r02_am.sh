#!/bin/bash
# round-2 (session 2): config 5 (ResNet-50 step, whole-step CUDA graph) at N=4 with the allreduce on 16/32 CTAs: FUSED vs PUSH vs NCCL
cd "$(dirname "$0")/../.."
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((28800+RANDOM%90)) "$@"; }
for m in push fused; do for nb in 16 32; do
  tr 4 tools/dp_resnet50.py --comm multiring --graph 1 --mode $m --nblocks $nb > gpurun_out/am_dp4_${m}_${nb}.jsonl 2>> gpurun_out/am.err
done; done
tr 4 tools/dp_resnet50.py --comm nccl --graph 1 > gpurun_out/am_dp4_nccl.jsonl 2>> gpurun_out/am.err
