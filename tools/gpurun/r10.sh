RBX_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 tools/latency_multi.py > gpurun_out/r10_latency2.log 2>&1
for tile in 256 512 1024 2048; do
RBX_TILE=$tile timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 tools/tune_multi.py --elems 1,262144,1048576,4194304,25600000 --nblocks 148 --threads 512 --modes fused > gpurun_out/r10_tune2_tile$tile.log 2>&1
done
for lt in 0 512 2048; do
RBX_LOCAL_TILE=$lt timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r10_bench1_lt$lt.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r10_virtual.log 2>&1; echo rc=$? >> gpurun_out/r10_virtual.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r10_multi.log 2>&1; echo rc=$? >> gpurun_out/r10_multi.log
