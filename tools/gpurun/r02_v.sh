#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 300 python tools/hostmem_probe.py --bufs 8 > gpurun_out/v_hostmem8.json 2> gpurun_out/v.err
timeout 300 python tools/hostmem_probe.py --bufs 1 > gpurun_out/v_hostmem1.json 2>> gpurun_out/v.err
