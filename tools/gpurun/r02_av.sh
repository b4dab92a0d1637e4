#!/bin/bash
# round-2 (session 2): ncu (full + Nvlink) of the final FUSED kernel in the 2-GPU harness, grid (2)
cd "$(dirname "$0")/../.."
timeout 300 python tools/fused_ncu.py --gpus 2 > gpurun_out/av_fused2_harness.json 2> gpurun_out/av.err
timeout 900 ncu --set full --section Nvlink --section Nvlink_Tables --clock-control none --import-source on -k regex:rbx_fused_kernel -c 2 -o gpurun_out/av_fused2 python tools/fused_ncu.py --gpus 2 --iters 1 > gpurun_out/av_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/av_ncu.log
ncu -i gpurun_out/av_fused2.ncu-rep --page raw --csv > gpurun_out/av_fused2_raw.csv 2>> gpurun_out/av.err
ncu -i gpurun_out/av_fused2.ncu-rep --page details --csv > gpurun_out/av_fused2_details.csv 2>> gpurun_out/av.err
