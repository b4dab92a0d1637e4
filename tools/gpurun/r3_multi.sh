./tools/nvlink_probe 51200000 > gpurun_out/r3_probe.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/r3_multi2.log 2>&1; echo rc=$? >> gpurun_out/r3_multi2.log
