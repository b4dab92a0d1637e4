#!/bin/bash
# round-2: PUSH through the matched-stage kernel -- parity, then PUSH vs FUSED by CTA count
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "all_decompositions or full_size or randomised" > gpurun_out/y_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/y_pytest.log
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((29000+RANDOM%90)) "$@"; }
tr 2 tools/tune_multi.py --elems 25600000,6553600 --modes fused,push --nblocks 16,32,64,148 --threads 512 > gpurun_out/y_tune2.txt 2>> gpurun_out/y.err
tr 4 tools/tune_multi.py --elems 25600000,6553600 --modes fused,push --nblocks 16,32,64,148 --threads 512 > gpurun_out/y_tune4.txt 2>> gpurun_out/y.err
RBX_PUSH_KERNEL=0 tr 4 tools/tune_multi.py --elems 25600000 --modes push --nblocks 32,148 --threads 512 > gpurun_out/y_tune4_push_generic.txt 2>> gpurun_out/y.err
