timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x > gpurun_out/r20_virtual.log 2>&1; echo rc=$? >> gpurun_out/r20_virtual.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r20_bench1.log 2>&1
RBX_LOCAL_GENERIC=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r20_bench1_generic.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --dtype bf16 > gpurun_out/r20_bench1_bf16.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r20_smoke.log 2>&1
