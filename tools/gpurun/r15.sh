T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for v in ld16 ld8; do
  if [ $v = ld8 ]; then export RBX_LIB_PATH=$PWD/paper_1708_02188_b200/librbx_ld8.so; else unset RBX_LIB_PATH; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r15_bench1_$v.log 2>&1
  timeout 300 $T --nproc-per-node 2 --master-port 29550 bench.py --gpus 2 --steps 20 --warmup 5 --no-nccl > gpurun_out/r15_bench2_$v.log 2>&1
done
unset RBX_LIB_PATH
timeout 300 $T --nproc-per-node 2 --master-port 29551 tools/nvlink_counters.py > gpurun_out/r15_nvlink_counters2.log 2>&1
nvidia-smi nvlink -h > gpurun_out/r15_smi_nvlink_help.txt 2>&1
nvidia-smi nvlink -gt d -i 0 > gpurun_out/r15_smi_nvlink_gt.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r15_virtual.log 2>&1; echo rc=$? >> gpurun_out/r15_virtual.log
