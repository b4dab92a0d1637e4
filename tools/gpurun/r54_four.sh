#!/bin/bash
# 4 GPUs: every execution mode at N=2 and N=4 with the current defaults (102.4 MB fp32)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for m in fused ring_dims fused_pull push; do
timeout 200 $T --nproc-per-node $n --master-port 2993$n bench.py --gpus $n --mode $m --no-nccl --curve 0 > gpurun_out/r54_b${n}_$m.log 2>&1
done; done
timeout 200 $T --nproc-per-node 4 --master-port 29940 bench.py --gpus 4 --dims 4 --mode ring_dims --no-nccl --curve 0 > gpurun_out/r54_b4_dims4_ring_dims.log 2>&1
timeout 200 $T --nproc-per-node 4 --master-port 29941 bench.py --gpus 4 --dims 4 --no-nccl --curve 0 > gpurun_out/r54_b4_dims4_auto.log 2>&1
