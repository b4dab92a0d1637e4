#!/bin/bash
# round-2: configs 3 (bf16), 4 (ResNet-101 buckets) and 5 (ResNet-50 step) with the specialised kernels
cd "$(dirname "$0")/../.."
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29800+RANDOM%100)) "$@"; }
for n in 2 4; do
  tr $n tools/buckets.py --iters 20 > gpurun_out/g_buckets_$n.jsonl 2>> gpurun_out/g.err
  RBX_PDL=0 tr $n tools/buckets.py --iters 20 > gpurun_out/g_buckets_${n}_nopdl.jsonl 2>> gpurun_out/g.err
done
timeout 900 python bench.py --gpus 2 --dtype bf16 --steps 20 --warmup 5 > gpurun_out/g_bench2_bf16.json 2>> gpurun_out/g.err
timeout 900 python bench.py --gpus 4 --dtype bf16 --steps 20 --warmup 5 > gpurun_out/g_bench4_bf16.json 2>> gpurun_out/g.err
tr 1 tools/dp_resnet50.py --comm none --graph 1 > gpurun_out/g_dp1.jsonl 2>> gpurun_out/g.err
for n in 2 4; do
  for c in multiring nccl; do tr $n tools/dp_resnet50.py --comm $c --graph 1 > gpurun_out/g_dp${n}_${c}.jsonl 2>> gpurun_out/g.err; done
done
