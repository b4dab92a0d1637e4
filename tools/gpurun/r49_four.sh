#!/bin/bash
# 4 GPUs: MultiringDataParallel parity test; config-5 steps at N=1/2/4 (eager / whole-step graph; CTAs per allreduce)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dp.py -q -x > gpurun_out/r49_dp_test.log 2>&1; echo rc=$? >> gpurun_out/r49_dp_test.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python tools/dp_resnet50.py --comm none --graph 0 > gpurun_out/r49_n1_eager.log 2>&1
timeout 300 python tools/dp_resnet50.py --comm none --graph 1 > gpurun_out/r49_n1_graph.log 2>&1
for n in 2 4; do
for nb in 8 16 32; do
timeout 300 $T --nproc-per-node $n --master-port 2976$n tools/dp_resnet50.py --comm multiring --graph 1 --nblocks $nb > gpurun_out/r49_n${n}_mr_graph_nb$nb.log 2>&1
done
timeout 300 $T --nproc-per-node $n --master-port 2977$n tools/dp_resnet50.py --comm multiring --graph 0 --nblocks 16 > gpurun_out/r49_n${n}_mr_eager_nb16.log 2>&1
timeout 300 $T --nproc-per-node $n --master-port 2978$n tools/dp_resnet50.py --comm nccl --graph 1 > gpurun_out/r49_n${n}_nccl_graph.log 2>&1
timeout 300 $T --nproc-per-node $n --master-port 2979$n tools/dp_resnet50.py --comm nccl --graph 0 > gpurun_out/r49_n${n}_nccl_eager.log 2>&1
timeout 300 $T --nproc-per-node $n --master-port 2980$n tools/ddp_resnet50.py --comm nccl --iters 30 > gpurun_out/r49_n${n}_ddp_nccl.log 2>&1
done
