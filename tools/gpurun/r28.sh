#!/bin/bash
# LL one-shot vs two-shot timelines + fair sweep (2 GPUs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for os in 0 65536; do
  RBX_LL_ONESHOT_BYTES=$os LAT_SIZES=1,1024,16384 LAT_MODES=ll RBX_TRACE=1 $T --master-port 29551 tools/latency_multi.py > gpurun_out/r28_latency_os$os.log 2>&1
done
$T --master-port 29552 tools/sweep.py --dtypes f32 --max-bytes 4194304 --iters 40 --out gpurun_out/r28_sweep2_auto.jsonl > gpurun_out/r28_sweep.log 2>&1
RBX_LL_ONESHOT_BYTES=0 $T --master-port 29553 tools/sweep.py --dtypes f32 --max-bytes 1048576 --iters 40 --mode ll --out gpurun_out/r28_sweep2_twoshot.jsonl >> gpurun_out/r28_sweep.log 2>&1
