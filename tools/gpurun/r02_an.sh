#!/bin/bash
# round-2 (session 2): reduce_scatter in PUSH / RING_DIMS through the matched-stage kernel: parity, then RS busbw by mode at N=2/4
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "reduce_scatter_allgather_pair" > gpurun_out/an_pytest.log 2>&1; echo rc=$? >> gpurun_out/an_pytest.log
tr() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=$((28800+RANDOM%90)) "$@"; }
tr 2 tools/tune_multi.py --elems 25600000,6553600 --ops reduce_scatter,allgather,allreduce --modes fused,push --nblocks 148 --threads 512 > gpurun_out/an_tune2.txt 2>> gpurun_out/an.err
tr 4 tools/tune_multi.py --elems 25600000,6553600 --ops reduce_scatter,allgather,allreduce --modes fused,push,ring_dims --nblocks 148 --threads 512 > gpurun_out/an_tune4.txt 2>> gpurun_out/an.err
# LL one-shot vs two-shot at N=2: device timelines (4 KB, 64 KB)
LAT_SIZES=1024,16384 LAT_MODES=ll RBX_TRACE=1 tr 2 tools/latency_multi.py > gpurun_out/an_lat_twoshot.jsonl 2>> gpurun_out/an.err
RBX_LL_ONESHOT_BYTES=65536 LAT_SIZES=1024,16384 LAT_MODES=ll RBX_TRACE=1 tr 2 tools/latency_multi.py > gpurun_out/an_lat_oneshot.jsonl 2>> gpurun_out/an.err
