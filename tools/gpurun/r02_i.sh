#!/bin/bash
# round-2: process exit with / without closing the communicator (and with a captured graph)
cd "$(dirname "$0")/../.."
tr() { timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$((29900+RANDOM%90)) "$@"; }
for c in 1 0; do for g in 0 1; do
  s=$(date +%s.%N); tr tools/exit_probe.py --close $c --graph $g > gpurun_out/i_exit_c${c}_g${g}.log 2>&1; rc=$?; e=$(date +%s.%N)
  echo "close=$c graph=$g rc=$rc wall=$(python3 -c "print(round($e-$s,1))")" >> gpurun_out/i_exit_summary.txt
done; done
s=$(date +%s.%N); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29991 tools/dp_resnet50.py --comm multiring --graph 1 > gpurun_out/i_dp2.jsonl 2> gpurun_out/i_dp2.err; rc=$?; e=$(date +%s.%N)
echo "dp_resnet50 multiring N=2 rc=$rc wall=$(python3 -c "print(round($e-$s,1))")" >> gpurun_out/i_exit_summary.txt
