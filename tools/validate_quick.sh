#!/bin/bash
# Short box validation: smoke, the GPU suite, N=1 and N=2 bench lines.
#   gpurun --gpus 2 --timeout 3000 -- 'bash tools/validate_quick.sh'
set -u
mkdir -p gpurun_out
S=gpurun_out/quick_summary.txt
: > $S
step() {
  local name=$1 secs=$2
  shift 2
  local t0=$(date +%s)
  timeout --kill-after=20 "$secs" bash -c "$*" > "gpurun_out/quick_${name}.log" 2>&1
  local rc=$?
  echo "$name rc=$rc $(( $(date +%s) - t0 ))s" | tee -a $S
  return $rc
}
step smoke 300 "python -c 'import __graft_entry__ as g; g.smoke()'"
step pytest_gpu 2100 "python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rfE"
step bench1 600 "python bench.py --steps 5 --warmup 3"
if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
  step bench2 900 "python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3"
fi
cat $S
