#!/bin/bash
# ncu evidence for the N=1 hot kernel (local reduce, config 2): launch list + one full capture.
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/r12_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r12_launches.csv $CMD > gpurun_out/r12_ncu_launches.log 2>&1
$CMD > gpurun_out/r12_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rbx_step -s 4 -c 1 -o gpurun_out/r12_prof_local $CMD > gpurun_out/r12_ncu_full.log 2>&1
echo done > gpurun_out/r12_done.txt
