#!/bin/bash
# round-2: the round-end driver sequence on one B200 (full GPU suite, smoke, N=1 bench) + the ncu launch list of the bench
cd "$(dirname "$0")/../.."
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/e_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/e_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/e_bench1.json 2> gpurun_out/e_bench1.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e_launches_n1.csv python bench.py --steps 20 --warmup 5 > gpurun_out/e_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/e_ncu.log
