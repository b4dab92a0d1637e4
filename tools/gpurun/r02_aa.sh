#!/bin/bash
# round-2: config 5 (ResNet-50 step, whole-step CUDA graph) with the allreduce on few SMs: FUSED vs PUSH
cd "$(dirname "$0")/../.."
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((28800+RANDOM%90)) "$@"; }
for n in 2 4; do
  for m in push fused; do for nb in 16 32; do
    tr $n tools/dp_resnet50.py --comm multiring --graph 1 --mode $m --nblocks $nb > gpurun_out/aa_dp${n}_${m}_${nb}.jsonl 2>> gpurun_out/aa.err
  done; done
  tr $n tools/dp_resnet50.py --comm nccl --graph 1 > gpurun_out/aa_dp${n}_nccl.jsonl 2>> gpurun_out/aa.err
done
tr 1 tools/dp_resnet50.py --comm none --graph 1 > gpurun_out/aa_dp1.jsonl 2>> gpurun_out/aa.err
