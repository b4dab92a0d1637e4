#!/bin/bash
# round-2 (session 2): LL kernel with a per-thread epoch read (no barrier before the first data loads): parity, then an A/B against the previous library at N=2, 4 KB-1 MB
cd "$(dirname "$0")/../.."
timeout 1200 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_multi.py -m gpu -q -x > gpurun_out/at_pytest.log 2>&1; echo rc=$? >> gpurun_out/at_pytest.log
tr() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$((28800+RANDOM%90)) "$@"; }
for rep in 1 2; do
  for lib in librbx.so librbx_old.so; do
    RBX_LIB_PATH=$PWD/paper_1708_02188_b200/$lib tr tools/sweep.py --max-bytes 1048576 --dtypes f32 --iters 40 --out gpurun_out/at_sweep_${lib%.so}_$rep.jsonl > /dev/null 2>> gpurun_out/at.err
  done
done
