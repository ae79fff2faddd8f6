#!/usr/bin/env bash
# ncu --set full of one warm K1 pass and one screened cold pass of a cfg3 bench step.
#   bash tools/ncu_warm.sh TAG
set -u
TAG=${1:-warm}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_lse_tq_kernelILb0ELb0E' -s 4 -c 1 -o "$OUT/k1_warm" \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > "$OUT/ncu_warm.log" 2>&1
echo "warm rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_lse_tq_kernelILb0ELb1E' -s 0 -c 1 -o "$OUT/k1_screen" \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > "$OUT/ncu_screen.log" 2>&1
echo "screen rc=$?"
ls -la "$OUT"
