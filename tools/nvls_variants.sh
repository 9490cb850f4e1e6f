#!/bin/bash
# NVLS loop variants at N GPUs: each variant in its own job.
W=${1:-4}
for v in 0 1 2 3; do
  echo "== variant $v"
  NEZHA_NVLS_VARIANT=$v python tools/rail_perf.py $W nvls:32,nvls:64 16777216,67108864,268435456,1073741824
done
