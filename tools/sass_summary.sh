#!/bin/bash
# Static kernel evidence, no GPU needed: per-kernel ptxas resources and the
# SASS instructions that prove each rail's data path compiled as designed.
#   bash tools/sass_summary.sh > profiles/r02/sass_summary.txt
# Run after `make -C paper_2405_17870_b200/csrc` (reads its ptxas logs and .o).
set -eu
cd "$(dirname "$0")/.."
OBJS="build/csrc/cuda/rails.cu.o build/csrc/cuda/rails_vr.cu.o"
LOG=$(mktemp)
SASS=$(mktemp)
trap 'rm -f "$SASS" "$LOG"' EXIT
for OBJ in $OBJS; do
  [ -f "$OBJ" ] && [ -f "$OBJ.ptxas.log" ] || { echo "build first: make -C paper_2405_17870_b200/csrc" >&2; exit 1; }
  cat "$OBJ.ptxas.log" >> "$LOG"
  cuobjdump -sass "$OBJ" >> "$SASS"
done

echo "# sm_100a static summary of $OBJS ($(git rev-parse --short HEAD 2>/dev/null || echo '?'))"
echo "# nvcc: $(nvcc --version | tail -1)"
echo
echo "## ptxas resources per kernel (registers | stack | spills)"
awk '/Function properties for/{f=$NF} /stack frame/{sf=$0} /Used [0-9]+ registers/{
       match($0, /Used [0-9]+ registers/); r=substr($0, RSTART+5, RLENGTH-15);
       gsub(/^ +/, "", sf); print f "\t" r " regs\t" sf }' "$LOG" | c++filt | sort
echo
echo "## kernels with spills"
awk '/Function properties for/{f=$NF} /spill stores/ && !/ 0 bytes spill stores, 0 bytes spill loads/{print f}' "$LOG" \
  | c++filt | sort || true
echo
echo "## data-path SASS per kernel family (instruction counts over all instances)"
echo "# LDGMC.* = multimem.ld_reduce (NVSwitch reduce, NVLS rail)"
echo "# LDL / STL = local memory (spills); the loopback *_vr grids select their rank's arguments by blockIdx.y"
echo "# LDG.E.NA.128 / STG.E.128* = 128-bit vectorised loads / peer stores"
awk '
  /Function :/ { fn = $3; next }
  /\/\*[0-9a-f]+\*\// {
    line = $0; sub(/^[ \t]*\/\*[0-9a-f]+\*\/[ \t]+/, "", line); sub(/ *;.*/, "", line)
    n = split(line, t, " "); op = t[1]; if (op ~ /^@/) op = t[2]
    if (op ~ /^(LDGMC|UBLKCP|UTMALDG|UTMASTG|SYNCS|LDG\.E.*128|STG\.E.*128|LDS\.128|STS\.128|SHFL|LDL|STL)/) c[fn "\t" op]++
  }
  END { for (k in c) print k "\t" c[k] }' "$SASS" | c++filt \
  | sed -E -e 's/^void nz::([a-z_]+)<[^\t]*/\1/' -e 's/^nz::([a-z_]+)\([^\t]*/\1/' \
  | awk -F'\t' '{s[$1 "\t" $2] += $3} END {for (k in s) print k "\t" s[k]}' | sort
