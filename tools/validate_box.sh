#!/bin/bash
# One gpurun call that validates the tree on a box (development aid).
#   gpurun --gpus 2 --timeout 2400 -- 'bash tools/validate_box.sh'
# Every step runs under its own timeout and logs to gpurun_out/val_*.log;
# a failing step does not stop the later ones. Summary: gpurun_out/val_summary.txt
set -u
mkdir -p gpurun_out
S=gpurun_out/val_summary.txt
: > $S
step() {  # step NAME SECONDS CMD...
  local name=$1 secs=$2
  shift 2
  local t0=$(date +%s)
  timeout --kill-after=20 "$secs" bash -c "$*" > "gpurun_out/val_${name}.log" 2>&1
  local rc=$?
  echo "$name rc=$rc $(( $(date +%s) - t0 ))s" | tee -a $S
  return $rc
}
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/val_gpus.csv 2>&1
step build 300 "python -c 'import __graft_entry__ as g; g.build()'"
step smoke 300 "python -c 'import __graft_entry__ as g; g.smoke()'"
step pytest_gpu 2400 "python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rfE"
step bench1 600 "python bench.py --steps 5 --warmup 3"
step copy_plain 300 "python tools/ncu_copy_n1.py" && \
  step ncu_copy 900 "ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 1 -c 1 -f -o gpurun_out/ncu_copy_n1 python tools/ncu_copy_n1.py"
if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
  step bench2 900 "python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3"
  step bench2x 900 "python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 5 --warmup 3 --tune --no-failover --no-e2e"
  step train2 900 "python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 tools/ddp_train_bench.py resnet50,bert 20"
  for v in "" "NEZHA_LL_MAX=0"; do
    step "smpaths_${#v}" 400 "$v python tools/rail_perf.py 2 sm 65536,262144,1048576,2097152,4194304,8388608"
  done
  for m in 0 1 2; do
    step pool$m 300 "python tools/run_spawn.py 2 tools/engine_hot_probe.py nvls,ce,sm 0.33 $m"
  done
fi
cat $S
