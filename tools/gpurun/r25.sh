#!/bin/bash
# small-message sweep with the host well ahead, latency timeline, DDP hook-cost isolation (2 GPUs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29521 tools/sweep.py --dtypes f32 --max-bytes 67108864 --out gpurun_out/r25_sweep2.jsonl > gpurun_out/r25_sweep.log 2>&1
RBX_TRACE=1 $T --master-port 29522 tools/latency_multi.py > gpurun_out/r25_latency.log 2>&1
for rep in 1 2; do
  for c in nccl nccl_hook ours; do
    $T --master-port 29523 tools/ddp_resnet50.py --comm $c --nblocks 16 >> gpurun_out/r25_ddp.jsonl 2>>gpurun_out/r25_ddp.err
  done
done
