#!/bin/bash
# prologue probe + current latency timeline + DDP nblocks sweep (2 GPUs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 ./tools/entry_probe > gpurun_out/r24_entry.txt 2>&1; echo "rc=$?" >> gpurun_out/r24_entry.txt
RBX_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/latency_multi.py > gpurun_out/r24_latency.log 2>&1
for nb in 8 16 32; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/ddp_resnet50.py --comm ours --nblocks $nb >> gpurun_out/r24_ddp.jsonl 2>>gpurun_out/r24_ddp.err
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/ddp_resnet50.py --comm nccl >> gpurun_out/r24_ddp.jsonl 2>>gpurun_out/r24_ddp.err
