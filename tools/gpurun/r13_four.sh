T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r13_bench1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r13_virtual.log 2>&1; echo rc=$? >> gpurun_out/r13_virtual.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r13_multi.log 2>&1; echo rc=$? >> gpurun_out/r13_multi.log
timeout 300 $T --nproc-per-node 4 --master-port 29520 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r13_bench4.log 2>&1
timeout 300 $T --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r13_bench2.log 2>&1
timeout 900 $T --nproc-per-node 4 --master-port 29522 tools/sweep.py --out gpurun_out/r13_sweep4.jsonl > gpurun_out/r13_sweep4.log 2>&1
timeout 300 $T --nproc-per-node 4 --master-port 29523 tools/buckets.py > gpurun_out/r13_buckets4.log 2>&1
timeout 300 $T --nproc-per-node 2 --master-port 29524 tools/buckets.py > gpurun_out/r13_buckets2.log 2>&1
timeout 300 python tools/ddp_resnet50.py > gpurun_out/r13_ddp1.log 2>&1
for n in 2 4; do for c in ours nccl; do
timeout 400 $T --nproc-per-node $n --master-port 2953$n tools/ddp_resnet50.py --comm $c > gpurun_out/r13_ddp${n}_$c.log 2>&1
done; done
