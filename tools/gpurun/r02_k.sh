#!/bin/bash
# round-2: graph replay vs direct launch; static vs dynamic tiles (fused kernel)
cd "$(dirname "$0")/../.."
tr() { n=$1; shift; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29600+RANDOM%90)) "$@"; }
for n in 2 4; do
  tr $n tools/graph_probe.py > gpurun_out/k_graph$n.jsonl 2>> gpurun_out/k.err
  RBX_PDL=0 tr $n tools/graph_probe.py > gpurun_out/k_graph${n}_nopdl.jsonl 2>> gpurun_out/k.err
  RBX_FUSED_DBG=16 timeout 600 python bench.py --gpus $n --steps 20 --warmup 5 --curve 0 --no-cpu-baseline --no-nccl > gpurun_out/k_bench${n}_static.json 2>> gpurun_out/k.err
  timeout 600 python bench.py --gpus $n --steps 20 --warmup 5 --curve 0 --no-cpu-baseline --no-nccl > gpurun_out/k_bench${n}_dyn.json 2>> gpurun_out/k.err
done
