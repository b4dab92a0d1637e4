./tools/flag_probe > gpurun_out/r9_flag_probe.txt 2>&1
./tools/local_probe > gpurun_out/r9_local_probe.txt 2>&1
