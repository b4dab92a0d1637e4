#!/bin/bash
# 4 GPUs: final validation (after per-step tiles, IPC refcount change): full GPU suite, smoke, bench + reference arms N=1/2/4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r61_gpu.log 2>&1; echo rc=$? >> gpurun_out/r61_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r61_smoke.log 2>&1; echo rc=$? >> gpurun_out/r61_smoke.log
timeout 300 python bench.py > gpurun_out/r61_bench1.log 2>&1
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r61_ref1.log 2>&1
for n in 2 4; do
timeout 300 $T --nproc-per-node $n --master-port 2991$n bench.py --gpus $n > gpurun_out/r61_bench$n.log 2>&1
timeout 300 $T --nproc-per-node $n --master-port 2992$n bench.py --impl reference --gpus $n --steps 5 --warmup 3 > gpurun_out/r61_ref$n.log 2>&1
done
