#!/bin/bash
# DDP ResNet-50 at N=2: where does the comm-hook gap come from (noop hook = hook machinery only)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for rep in 1 2; do
  for c in nccl noop_hook nccl_hook ours; do
    $T --master-port 29601 tools/ddp_resnet50.py --comm $c --nblocks 16 --iters 30 >> gpurun_out/r35_ddp.jsonl 2>>gpurun_out/r35_ddp.err
  done
done
