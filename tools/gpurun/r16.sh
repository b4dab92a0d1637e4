#!/bin/bash
CMD="python tools/nvlink_ncu.py --iters 5"
$CMD > gpurun_out/r16_plain.log 2>&1 && \
ncu --set full --section Nvlink --section Nvlink_Tables --clock-control none -k regex:rbx_step -s 2 -c 1 -o gpurun_out/r16_prof_nvlink $CMD > gpurun_out/r16_ncu.log 2>&1
python tools/nvlink_ncu.py --iters 20 > gpurun_out/r16_nvlink_harness.log 2>&1
echo done > gpurun_out/r16_done.txt
