#!/bin/bash
# Probe: NVLink throughput counters around a command (wire-byte evidence).
nvidia-smi nvlink -gt d -i 0 > gpurun_out/nvl_before.txt 2>&1
"$@"
nvidia-smi nvlink -gt d -i 0 > gpurun_out/nvl_after.txt 2>&1
head -40 gpurun_out/nvl_after.txt
