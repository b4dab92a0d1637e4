#!/bin/bash
# round-2: CTA-count sweep of the fused kernel (SMs the collective needs) and host-pipeline windows at N=2
cd "$(dirname "$0")/../.."
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29400+RANDOM%90)) "$@"; }
tr 2 tools/tune_multi.py --elems 25600000,6553600 --modes fused --nblocks 16,32,48,64,96,148 --threads 512 > gpurun_out/n_tune2.jsonl 2>> gpurun_out/n.err
tr 4 tools/tune_multi.py --elems 25600000,6553600 --modes fused,ring_dims --nblocks 16,32,48,64,96,148 --threads 512 > gpurun_out/n_tune4.jsonl 2>> gpurun_out/n.err
for w in 8 16 64; do
  RBX_HOST_WINDOWS=$w timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --curve 0 --no-nccl --no-cpu-baseline > gpurun_out/n_bench2_w$w.json 2>> gpurun_out/n.err
done
