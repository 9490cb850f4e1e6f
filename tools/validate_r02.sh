#!/bin/bash
# Round-2 hardware re-entry ladder (after the round-1 NVLink incident), one
# GPU first. Every step has its own timeout and log; a failing step does not
# stop the later ones. Summary: gpurun_out/r02_summary.txt
#   gpurun --timeout 3000 -- 'bash tools/validate_r02.sh'          (1 GPU)
#   gpurun --gpus 2 --timeout 3000 -- 'NEZHA_DISABLE_MULTICAST=1 bash tools/validate_r02.sh multi'
set -u
mkdir -p gpurun_out
S=gpurun_out/r02_summary.txt
: > $S
step() {  # step NAME SECONDS CMD...
  local name=$1 secs=$2
  shift 2
  local t0=$(date +%s)
  timeout --kill-after=20 "$secs" bash -c "$*" > "gpurun_out/r02_${name}.log" 2>&1
  local rc=$?
  echo "$name rc=$rc $(( $(date +%s) - t0 ))s" | tee -a $S
  return $rc
}
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_gpus.csv 2>&1
step smoke 600 "python -c 'import __graft_entry__ as g; g.smoke()'"
step loopback 2400 "python -m pytest tests/test_gpu_vranks.py -m gpu -q -p no:cacheprovider --timeout 900 -rfE -x"
step single 900 "python -m pytest tests/test_gpu_rails.py tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider --timeout 600 -rfE"
step bench1 900 "python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench1.json"
step launches 900 "ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python tools/ncu_loopback.py 8 4"
step ncu_fold 1500 "ncu --set full --clock-control none --import-source on -k regex:fold_kernel_vr -s 2 -c 1 -f -o gpurun_out/r02_ncu_fold_vr python tools/ncu_loopback.py 8 4"
step memcheck 1500 "compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_vranks.py -m gpu -q -p no:cacheprovider -k 'rails_bit_exact and 4'"
if [ "${1:-}" = "multi" ] && [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
  step rails2 900 "python -m pytest tests/test_gpu_rails.py -m gpu -q -p no:cacheprovider --timeout 600 -rfE -k 'multi_gpu and 2'"
  step engine2 1500 "python -m pytest tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider --timeout 900 -rfE"
  step bench2 900 "python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 10 --warmup 3 --latency-ops 2000 > gpurun_out/r02_bench2.json"
fi
cat $S
