set -x
nvidia-smi topo -m > gpurun_out/r2_topo.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r2_multi2.log 2>&1; echo rc=$? >> gpurun_out/r2_multi2.log
for mode in auto fused_pull ring_dims; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 --mode $mode > gpurun_out/r2_bench2_$mode.log 2>&1
done
