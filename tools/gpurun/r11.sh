RBX_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 tools/latency_multi.py > gpurun_out/r11_latency2.log 2>&1
for lt in 2048 4096 8192 32768; do
RBX_LOCAL_TILE=$lt timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r11_bench1_lt$lt.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 tools/sweep.py --out gpurun_out/r11_sweep2.jsonl > gpurun_out/r11_sweep2.log 2>&1
