#!/bin/bash
# round-2 (session 2): final code on ONE B200 as the driver runs it: whole GPU suite, smoke, bench N=1, reference arm; ncu launch list of the bench
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ao_pytest.log 2>&1; echo rc=$? >> gpurun_out/ao_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ao_smoke.log 2>&1; echo rc=$? >> gpurun_out/ao_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/ao_bench1.json 2> gpurun_out/ao_bench1.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ao_ref1.json 2> gpurun_out/ao_ref1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ao_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ao_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ao_ncu.log
