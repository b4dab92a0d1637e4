T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ddp.py -q > gpurun_out/r22_multi.log 2>&1; echo rc=$? >> gpurun_out/r22_multi.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r22_bench1.log 2>&1
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r22_ref1.log 2>&1
for n in 2 4; do
timeout 300 $T --nproc-per-node $n --master-port 2958$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r22_bench$n.log 2>&1
timeout 300 $T --nproc-per-node $n --master-port 2959$n bench.py --impl reference --gpus $n --steps 5 --warmup 3 > gpurun_out/r22_ref$n.log 2>&1
done
timeout 300 $T --nproc-per-node 4 --master-port 29600 bench.py --gpus 4 --steps 20 --warmup 5 --mode ring_dims --no-nccl > gpurun_out/r22_bench4_ringdims.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29601 tools/sweep.py --out gpurun_out/r22_sweep4.jsonl > gpurun_out/r22_sweep4.log 2>&1
timeout 300 $T --nproc-per-node 4 --master-port 29602 tools/buckets.py > gpurun_out/r22_buckets4.log 2>&1
timeout 400 $T --nproc-per-node 4 --master-port 29603 tools/ddp_resnet50.py --comm nccl > gpurun_out/r22_ddp4_nccl.log 2>&1
timeout 400 $T --nproc-per-node 4 --master-port 29604 tools/ddp_resnet50.py --comm ours > gpurun_out/r22_ddp4_ours.log 2>&1
timeout 300 python tools/ddp_resnet50.py > gpurun_out/r22_ddp1.log 2>&1
