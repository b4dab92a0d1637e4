#!/bin/bash
# DDP hook host cost (slow vs cached fast path) and the DDP step with the fast hook
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29621 tools/hook_overhead.py > gpurun_out/r37_hook.log 2>&1
for rep in 1 2; do
  for c in nccl ours; do
    $T --master-port 29622 tools/ddp_resnet50.py --comm $c --nblocks 16 --iters 30 >> gpurun_out/r37_ddp.jsonl 2>>gpurun_out/r37_ddp.err
  done
done
timeout 600 python -m pytest tests/test_gpu_ddp.py -q > gpurun_out/r37_pytest_ddp.log 2>&1; echo rc=$? >> gpurun_out/r37_pytest_ddp.log
