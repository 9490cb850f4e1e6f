#!/bin/bash
# Host-logic harness (tests/fakecuda) under ThreadSanitizer or
# AddressSanitizer: the product's host sources rebuilt with the sanitizer
# (kernels as PTX only), linked against the harness with its protocol
# restatements of the kernels (FAKECUDA_NO_SIMT: the sanitizers do not follow
# the SIMT stand-in's fiber stack switches), then a loopback engine run with
# an unplanned failover and readmit.
#   bash tools/harness_sanitize.sh tsan|asan
# TSan's expected reports: the failure monitor's volatile reads of the
# host-mapped launch status (written by the "device"); anything else is a
# host-side race.
set -eu
SAN=${1:-tsan}
FLAG=$([ "$SAN" = tsan ] && echo -fsanitize=thread || echo -fsanitize=address)
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/tests/fakecuda/build/$SAN
CU=/usr/local/cuda
mkdir -p $OUT/host $OUT/cuda
cd $ROOT/paper_2405_17870_b200/csrc
INC="-I$ROOT/include -I$CU/include -Icuda"
for f in host/*.cpp cuda/*.cpp; do
  /usr/bin/g++ -std=c++20 -O1 -g -fPIC $FLAG -ffp-contract=off $INC -c $f -o $OUT/${f%.cpp}.o &
done
for f in cuda/rails.cu cuda/rails_vr.cu; do
  $CU/bin/nvcc -std=c++20 -O1 -g -gencode arch=compute_100a,code=compute_100a \
    -Xcompiler -fPIC,$FLAG,-ffp-contract=off --expt-relaxed-constexpr $INC -c $f -o $OUT/$f.o &
done
wait
cd $ROOT/tests/fakecuda
for f in fakecuda emu_kernels; do
  /usr/bin/g++ -std=c++20 -O1 -g -fPIC $FLAG -DFAKECUDA_NO_SIMT -I$ROOT/include -I$CU/include -I$ROOT/paper_2405_17870_b200/csrc/cuda -I. \
    -c $f.cpp -o $OUT/$f.o
done
/usr/bin/g++ -shared $FLAG -Wl,-Bsymbolic -o $OUT/libnezha_b200_hostharness.so $OUT/fakecuda.o $OUT/emu_kernels.o \
  $OUT/host/*.o $OUT/cuda/*.o -lpthread -ldl -lrt
cd $ROOT
RT=$(gcc -print-file-name=lib$([ "$SAN" = tsan ] && echo tsan || echo asan).so)
export NEZHA_TEST_HOST_HARNESS_LIB=$OUT/libnezha_b200_hostharness.so NEZHA_DETECT_US=2000000 NEZHA_WATCHDOG_MS=5000
export TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0" ASAN_OPTIONS="detect_leaks=0"
LD_PRELOAD=$RT python - <<'PY'
import sys
sys.path.insert(0, ".")
import tests.test_gpu_vranks as T
from paper_2405_17870_b200 import run_ranks
from tests.workers import engine_worker
spec = {"rails": T.KINDS3, "rails_toml": T.TOML_LOOP, "sync_overhead_us": 0.0, "readmit_hold_us": 100000,
        "cases": [{"dtype": "f32", "nbytes": 4 << 20, "reps": 2},
                  {"dtype": "bf16", "nbytes": 8 << 20, "reps": 2, "fail": [2, 1], "fail_rep": 1},
                  {"dtype": "f32", "nbytes": (1 << 20) + 4, "reps": 1, "host": True},
                  {"dtype": "i32", "nbytes": 2 << 20, "reps": 1, "readmit": True}]}
res = run_ranks(2, lambda comm: engine_worker.run(comm, spec), timeout=900)
assert all(r["mismatch"] == 0 for rk in res for r in rk["results"])
print("harness run ok")
PY
