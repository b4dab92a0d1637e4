#!/bin/bash
# round-2: RING_DIMS kernel parity (4 GPUs) and RING_DIMS vs FUSED at (2,2), (4,), (2,)
cd "$(dirname "$0")/../.."
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -x > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest.log
for m in fused ring_dims; do
  timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 --curve 0 --no-cpu-baseline --no-nccl --mode $m > gpurun_out/f_bench4_$m.json 2>> gpurun_out/f_bench.err
  timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 --curve 0 --no-cpu-baseline --no-nccl --mode $m > gpurun_out/f_bench2_$m.json 2>> gpurun_out/f_bench.err
done
RBX_RINGS_KERNEL=0 timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 --curve 0 --no-cpu-baseline --no-nccl --mode ring_dims > gpurun_out/f_bench4_ring_dims_generic.json 2>> gpurun_out/f_bench.err
