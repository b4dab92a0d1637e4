#!/bin/bash
# round-2: PUSH with per-CTA rotated scatter -- parity + CTA sweep at N=4 (and N=2)
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "all_decompositions or randomised" > gpurun_out/z_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/z_pytest.log
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((28900+RANDOM%90)) "$@"; }
tr 4 tools/tune_multi.py --elems 25600000,6553600 --modes fused,push --nblocks 16,32,64,148 --threads 512 > gpurun_out/z_tune4.txt 2>> gpurun_out/z.err
tr 2 tools/tune_multi.py --elems 25600000,6553600 --modes push --nblocks 16,32,148 --threads 512 > gpurun_out/z_tune2.txt 2>> gpurun_out/z.err
