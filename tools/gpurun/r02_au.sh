#!/bin/bash
# round-2 (session 2): final code, whole GPU suite on one B200 + smoke + bench N=1
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/au_pytest.log 2>&1; echo rc=$? >> gpurun_out/au_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/au_smoke.log 2>&1; echo rc=$? >> gpurun_out/au_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/au_bench1.json 2> gpurun_out/au_bench1.err
