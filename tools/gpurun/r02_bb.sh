#!/bin/bash
# round-2 (session 2): rbx_comm_last_kernel -- every call takes the kernel the design says (worlds 2/4, ranks sharing one GPU)
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "specialised_kernels" > gpurun_out/bb_pytest.log 2>&1; echo rc=$? >> gpurun_out/bb_pytest.log
timeout 600 python -m pytest tests/test_gpu_virtual.py -m gpu -q -x -k "allreduce_host or all_decompositions" >> gpurun_out/bb_pytest.log 2>&1; echo rc=$? >> gpurun_out/bb_pytest.log
