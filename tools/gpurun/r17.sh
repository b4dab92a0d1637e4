T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r17_virtual.log 2>&1; echo rc=$? >> gpurun_out/r17_virtual.log
for lt in 512 1024 2048 4096; do
RBX_LOCAL_TILE=$lt timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r17_bench1_lt$lt.log 2>&1
done
for tile in 512 1024 2048; do
RBX_TILE=$tile timeout 600 $T --nproc-per-node 2 --master-port 29560 tools/tune_multi.py --elems 1048576,4194304,25600000 --nblocks 148 --threads 512 --modes fused > gpurun_out/r17_tune2_tile$tile.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r17_multi.log 2>&1; echo rc=$? >> gpurun_out/r17_multi.log
