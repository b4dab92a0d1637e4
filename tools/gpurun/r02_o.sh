#!/bin/bash
# round-2: config 3 size sweep (fp32 + bf16) at N=2/4 vs NCCL with the specialised kernels; smoke
cd "$(dirname "$0")/../.."
tr() { n=$1; shift; timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29300+RANDOM%90)) "$@"; }
tr 2 tools/sweep.py --iters 12 > gpurun_out/o_sweep2.jsonl 2>> gpurun_out/o.err
tr 4 tools/sweep.py --iters 12 > gpurun_out/o_sweep4.jsonl 2>> gpurun_out/o.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/o_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/o_smoke.log
