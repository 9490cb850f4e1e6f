#!/bin/bash
# compute-sanitizer memcheck over the single-GPU kernel tests (emulated rail
# folds, golden vectors, the loopback rails). One sanitizer per gpurun call:
#   gpurun --timeout 1800 -- 'bash tools/sanitize.sh'
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
  python -m pytest tests/test_gpu_rails.py tests/test_gpu_vranks.py -m gpu -q -p no:cacheprovider \
  -k "emulated or golden or config1 or (rails_bit_exact and 4)" > gpurun_out/sanitize.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize.log
tail -5 gpurun_out/sanitize.log
