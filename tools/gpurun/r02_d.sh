#!/bin/bash
# round-2: what makes the fused kernel's completion slow (device-clock brackets, n=1)
cd "$(dirname "$0")/../.."
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$1 tools/gap_probe.py; }
export GAP_SIZES=1,25600000
for v in 0 1 2 3 4 11; do RBX_FUSED_DBG=$v run $((29700+v)) > gpurun_out/d_gap_dbg$v.jsonl 2>> gpurun_out/d_gap.err; done
RBX_PLAIN_LAUNCH=1 run 29720 > gpurun_out/d_gap_plain.jsonl 2>> gpurun_out/d_gap.err
RBX_FUSED_KERNEL=0 run 29721 > gpurun_out/d_gap_generic.jsonl 2>> gpurun_out/d_gap.err
GAP_MODE=ll GAP_SIZES=1 run 29722 > gpurun_out/d_gap_ll.jsonl 2>> gpurun_out/d_gap.err
