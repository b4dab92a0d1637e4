#!/bin/bash
# smoke + default bench N=1 / N=2 with the host bound to the GPU's NUMA cores
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r40_smoke.log 2>&1; echo rc=$? >> gpurun_out/r40_smoke.log
timeout 300 python bench.py > gpurun_out/r40_bench1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 2 > gpurun_out/r40_bench2.log 2>&1
nvidia-smi topo -m > gpurun_out/r40_topo.txt 2>&1
