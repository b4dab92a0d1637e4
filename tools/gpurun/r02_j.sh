#!/bin/bash
# round-2: N=4 bench line (graph replay, PDL in LL), N=8 functional on 4 GPUs, reference arm at N=8, DDP hook config 5
cd "$(dirname "$0")/../.."
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/j_bench4.json 2> gpurun_out/j.err
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/j_bench2.json 2>> gpurun_out/j.err
timeout 1200 python bench.py --gpus 8 --steps 5 --warmup 3 > gpurun_out/j_bench8_shared.json 2>> gpurun_out/j.err
timeout 600 python bench.py --impl reference --gpus 8 --steps 5 --warmup 3 > gpurun_out/j_ref8.json 2>> gpurun_out/j.err
tr() { n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29700+RANDOM%90)) "$@"; }
for n in 2 4; do for c in ours nccl; do tr $n tools/ddp_resnet50.py --comm $c > gpurun_out/j_ddp${n}_$c.jsonl 2>> gpurun_out/j.err; done; done
