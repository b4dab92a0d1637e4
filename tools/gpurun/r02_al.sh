#!/bin/bash
# round-2 (session 2): ncu (full + Nvlink sections) of the product FUSED kernel in the single-process 4-GPU harness, grid (2,2)
cd "$(dirname "$0")/../.."
timeout 300 python tools/fused_ncu.py --gpus 4 > gpurun_out/al_fused4_harness.json 2> gpurun_out/al.err
timeout 1200 ncu --set full --section Nvlink --section Nvlink_Tables --clock-control none --import-source on -k regex:rbx_fused_kernel -c 4 -o gpurun_out/al_fused4 python tools/fused_ncu.py --gpus 4 --iters 1 > gpurun_out/al_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/al_ncu.log
ncu -i gpurun_out/al_fused4.ncu-rep --page raw --csv > gpurun_out/al_fused4_raw.csv 2>> gpurun_out/al.err
ncu -i gpurun_out/al_fused4.ncu-rep --page details --csv > gpurun_out/al_fused4_details.csv 2>> gpurun_out/al.err
