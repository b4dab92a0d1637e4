T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_ddp.py tests/test_gpu_virtual.py -q -x -k "ddp or graph" > gpurun_out/r14_ddp_graph_tests.log 2>&1; echo rc=$? >> gpurun_out/r14_ddp_graph_tests.log
timeout 300 $T --nproc-per-node 2 --master-port 29540 tools/nvlink_counters.py > gpurun_out/r14_nvlink_counters2.log 2>&1
timeout 300 $T --nproc-per-node 2 --master-port 29541 tools/nvlink_counters.py --mode ring_dims > gpurun_out/r14_nvlink_counters2_rd.log 2>&1
timeout 400 $T --nproc-per-node 2 --master-port 29542 tools/ddp_resnet50.py --comm nccl > gpurun_out/r14_ddp2_nccl.log 2>&1
for nb in 16 32 64 148; do
timeout 400 $T --nproc-per-node 2 --master-port 29543 tools/ddp_resnet50.py --comm ours --nblocks $nb > gpurun_out/r14_ddp2_ours_nb$nb.log 2>&1
done
