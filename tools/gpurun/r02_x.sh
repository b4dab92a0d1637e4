#!/bin/bash
# round-2: per-SM NVLink throughput with few CTAs: SM loads/stores vs TMA bulk
cd "$(dirname "$0")/../.."
PROBE_FEW_CTAS=1 tools/nvlink_ceiling 2 256 > gpurun_out/x_few2.jsonl 2> gpurun_out/x.err
