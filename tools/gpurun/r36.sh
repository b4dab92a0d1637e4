#!/bin/bash
# DDP overlap: CTA footprint of our kernels while they wait for the peer (registers block co-residency)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29611 tools/ddp_resnet50.py --comm nccl --iters 30 >> gpurun_out/r36_ddp.jsonl 2>>gpurun_out/r36_ddp.err
for cfg in "8 512" "4 512" "16 256" "8 256" "16 128" "32 128"; do
  set -- $cfg
  $T --master-port 29611 tools/ddp_resnet50.py --comm ours --nblocks $1 --threads $2 --iters 30 >> gpurun_out/r36_ddp.jsonl 2>>gpurun_out/r36_ddp.err
done
$T --master-port 29611 tools/ddp_resnet50.py --comm nccl --iters 30 >> gpurun_out/r36_ddp.jsonl 2>>gpurun_out/r36_ddp.err
