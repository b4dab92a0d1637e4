#!/bin/bash
# 4 GPUs: full GPU suite with dynamic tiles + pass_tile defaults, bench/reference arms N=1/2/4,
# sweeps and config-4 buckets at N=2/4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r46_gpu.log 2>&1; echo rc=$? >> gpurun_out/r46_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r46_smoke.log 2>&1; echo rc=$? >> gpurun_out/r46_smoke.log
timeout 300 python bench.py > gpurun_out/r46_bench1.log 2>&1
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r46_ref1.log 2>&1
for n in 2 4; do
timeout 300 $T --nproc-per-node $n --master-port 2981$n bench.py --gpus $n > gpurun_out/r46_bench$n.log 2>&1
timeout 300 $T --nproc-per-node $n --master-port 2982$n bench.py --impl reference --gpus $n --steps 5 --warmup 3 > gpurun_out/r46_ref$n.log 2>&1
RBX_TILE=2048 timeout 300 $T --nproc-per-node $n --master-port 2983$n bench.py --gpus $n --no-nccl > gpurun_out/r46_bench${n}_t2048.log 2>&1
timeout 1200 $T --nproc-per-node $n --master-port 2984$n tools/sweep.py --iters 20 --out gpurun_out/r46_sweep$n.jsonl > gpurun_out/r46_sweep$n.log 2>&1
timeout 300 $T --nproc-per-node $n --master-port 2985$n tools/buckets.py > gpurun_out/r46_buckets$n.log 2>&1
done
