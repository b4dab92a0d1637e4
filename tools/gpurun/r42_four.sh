#!/bin/bash
# 4 GPUs: re-verify HEAD (smoke, bench N=1/2/4), PCIe ceiling for the e2e leg
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r42_topo.txt 2>&1
lscpu > gpurun_out/r42_lscpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r42_smoke.log 2>&1; echo rc=$? >> gpurun_out/r42_smoke.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python tools/pcie_probe.py > gpurun_out/r42_pcie1.jsonl 2>&1
timeout 300 python tools/pcie_probe.py --no-bind > gpurun_out/r42_pcie1_nobind.jsonl 2>&1
timeout 300 $T --nproc-per-node 2 --master-port 29701 tools/pcie_probe.py > gpurun_out/r42_pcie2.jsonl 2>&1
timeout 300 $T --nproc-per-node 4 --master-port 29702 tools/pcie_probe.py > gpurun_out/r42_pcie4.jsonl 2>&1
timeout 300 python bench.py > gpurun_out/r42_bench1.log 2>&1
timeout 300 python bench.py --e2e-chunks 32 --no-cpu-baseline > gpurun_out/r42_bench1_c32.log 2>&1
timeout 300 $T --nproc-per-node 2 --master-port 29703 bench.py --gpus 2 > gpurun_out/r42_bench2.log 2>&1
timeout 300 $T --nproc-per-node 2 --master-port 29704 bench.py --gpus 2 --e2e-chunks 32 --no-nccl > gpurun_out/r42_bench2_c32.log 2>&1
timeout 300 $T --nproc-per-node 4 --master-port 29705 bench.py --gpus 4 > gpurun_out/r42_bench4.log 2>&1
timeout 300 $T --nproc-per-node 4 --master-port 29706 bench.py --gpus 4 --e2e-chunks 32 --no-nccl > gpurun_out/r42_bench4_c32.log 2>&1
