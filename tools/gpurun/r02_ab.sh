#!/bin/bash
# round-2 (session 2): HEAD state on one GPU, as the driver runs it: GPU suite, smoke, bench N=1, reference arm
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ab_pytest.log 2>&1; echo rc=$? >> gpurun_out/ab_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ab_smoke.log 2>&1; echo rc=$? >> gpurun_out/ab_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/ab_bench1.json 2> gpurun_out/ab_bench1.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ab_ref1.json 2> gpurun_out/ab_ref1.err
