timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r6_virtual.log 2>&1; echo rc=$? >> gpurun_out/r6_virtual.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r6_multi.log 2>&1; echo rc=$? >> gpurun_out/r6_multi.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r6_bench1.log 2>&1
for tile in 0 1024 4096 16384; do
RBX_TILE=$tile timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 tools/tune_multi.py --elems 262144,1048576,25600000 --nblocks 148 --threads 512 > gpurun_out/r6_tune2_tile$tile.log 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r6_bench2.log 2>&1
