#!/bin/bash
# round-2: the driver's round-end sequence on one B200 after the last kernel changes
cd "$(dirname "$0")/../.."
timeout 2700 python -m pytest tests -m gpu -q -rs --durations=20 > gpurun_out/l_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/l_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/l_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/l_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/l_bench1.json 2> gpurun_out/l_bench1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/l_ref1.json 2>> gpurun_out/l_bench1.err
