timeout 1200 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/r4_multi2.log 2>&1; echo rc=$? >> gpurun_out/r4_multi2.log
timeout 600 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r4_virtual.log 2>&1; echo rc=$? >> gpurun_out/r4_virtual.log
