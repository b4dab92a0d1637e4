T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r23_virtual.log 2>&1; echo rc=$? >> gpurun_out/r23_virtual.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "bf16 or decompositions" > gpurun_out/r23_multi.log 2>&1; echo rc=$? >> gpurun_out/r23_multi.log
