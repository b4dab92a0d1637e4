T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r19_virtual.log 2>&1; echo rc=$? >> gpurun_out/r19_virtual.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r19_multi.log 2>&1; echo rc=$? >> gpurun_out/r19_multi.log
timeout 600 $T --nproc-per-node 2 --master-port 29570 tools/tune_multi.py --elems 1,262144,1048576,4194304,25600000,268435456 --nblocks 148 --threads 512 --modes fused,push > gpurun_out/r19_tune2.log 2>&1
for mode in fused push; do
timeout 300 $T --nproc-per-node 2 --master-port 29571 bench.py --gpus 2 --steps 20 --warmup 5 --mode $mode > gpurun_out/r19_bench2_$mode.log 2>&1
done
