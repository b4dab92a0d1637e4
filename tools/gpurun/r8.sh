./tools/local_probe > gpurun_out/r8_local_probe.txt 2>&1
RBX_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 tools/latency_multi.py > gpurun_out/r8_latency2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r8_virtual.log 2>&1; echo rc=$? >> gpurun_out/r8_virtual.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r8_multi.log 2>&1; echo rc=$? >> gpurun_out/r8_multi.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r8_bench1.log 2>&1
