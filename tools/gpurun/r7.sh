timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r7_virtual.log 2>&1; echo rc=$? >> gpurun_out/r7_virtual.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r7_multi.log 2>&1; echo rc=$? >> gpurun_out/r7_multi.log
for bpc in 131072 524288 2097152; do
RBX_BYTES_PER_CTA=$bpc timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 tools/tune_multi.py --elems 1,65536,262144,1048576,4194304,25600000 --nblocks 148 --threads 512 --modes fused,ring_dims > gpurun_out/r7_tune2_bpc$bpc.log 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r7_bench2.log 2>&1
