#!/bin/bash
# 2 GPUs: MultiringDataParallel parity test + config-5 step times (eager / whole-step graph) vs DDP+NCCL
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dp.py -q -x > gpurun_out/r48_dp_test.log 2>&1; echo rc=$? >> gpurun_out/r48_dp_test.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 300 python tools/dp_resnet50.py --comm none --graph 0 > gpurun_out/r48_n1_eager.log 2>&1
timeout 300 python tools/dp_resnet50.py --comm none --graph 1 > gpurun_out/r48_n1_graph.log 2>&1
timeout 300 $T --master-port 29751 tools/dp_resnet50.py --comm multiring --graph 0 > gpurun_out/r48_n2_mr_eager.log 2>&1
timeout 300 $T --master-port 29752 tools/dp_resnet50.py --comm multiring --graph 1 > gpurun_out/r48_n2_mr_graph.log 2>&1
timeout 300 $T --master-port 29753 tools/dp_resnet50.py --comm nccl --graph 0 > gpurun_out/r48_n2_nccl_eager.log 2>&1
timeout 300 $T --master-port 29754 tools/dp_resnet50.py --comm nccl --graph 1 > gpurun_out/r48_n2_nccl_graph.log 2>&1
timeout 300 $T --master-port 29755 tools/ddp_resnet50.py --comm nccl --iters 30 > gpurun_out/r48_n2_ddp_nccl.log 2>&1
