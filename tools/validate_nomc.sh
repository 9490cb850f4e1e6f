#!/bin/bash
# Cautious first multi-GPU call after the NVLink incident: no NVSwitch
# multicast at all (NEZHA_DISABLE_MULTICAST=1: no NVLS rail, no multicast
# binding), only unicast peer loads/stores and copy-engine DMA.
#   gpurun --gpus 2 --timeout 2400 -- 'bash tools/validate_nomc.sh'
set -u
mkdir -p gpurun_out
export NEZHA_DISABLE_MULTICAST=1
S=gpurun_out/nomc_summary.txt
: > $S
step() {
  local name=$1 secs=$2
  shift 2
  local t0=$(date +%s)
  timeout --kill-after=20 "$secs" bash -c "$*" > "gpurun_out/nomc_${name}.log" 2>&1
  local rc=$?
  echo "$name rc=$rc $(( $(date +%s) - t0 ))s" | tee -a $S
  return $rc
}
step smoke 300 "python -c 'import __graft_entry__ as g; g.smoke()'"
step single_gpu 900 "python -m pytest tests/test_gpu_rails.py tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider --timeout 600 -rfE -k 'emulated or golden or config1 or single_gpu'"
step rails 600 "python tools/run_spawn.py 2 tests/workers/rail_worker.py \"\$(python -c 'import json,sys; sys.path.insert(0,\".\"); from tests.test_gpu_rails import MULTI, random_rail_cases; print(json.dumps([c for c in MULTI + random_rail_cases(102) if c[\"kind\"] != \"nvls\"]))')\""
step engine 600 "python tools/run_spawn.py 2 tests/workers/engine_worker.py '{\"rails\": [\"ce\", \"sm\"], \"calibrate_max_bytes\": 67108864, \"cases\": [{\"dtype\": \"f32\", \"nbytes\": 67108864, \"reps\": 3}, {\"dtype\": \"bf16\", \"nbytes\": 3000002, \"reps\": 2}, {\"dtype\": \"i32\", \"nbytes\": 8192, \"reps\": 2, \"host\": true}, {\"dtype\": \"f32\", \"nbytes\": 41943044, \"reps\": 1, \"device\": true}, {\"dtype\": \"bf16\", \"nbytes\": 268435456, \"reps\": 2, \"fail\": [1, 3], \"fail_rep\": 1}]}'"
step bench2 900 "python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --rails ce,sm"
cat $S
