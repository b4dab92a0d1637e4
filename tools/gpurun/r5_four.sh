nvidia-smi topo -m > gpurun_out/r5_topo.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/r5_multi4.log 2>&1; echo rc=$? >> gpurun_out/r5_multi4.log
for mode in auto ring_dims; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 20 --warmup 5 --mode $mode > gpurun_out/r5_bench4_$mode.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 tools/tune_multi.py --elems 1048576,25600000 > gpurun_out/r5_tune4.log 2>&1
