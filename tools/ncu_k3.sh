#!/usr/bin/env bash
# ncu --set full of the gradient's transport kernel (K3) in a cfg3 bench step.
set -u
TAG=${1:-k3}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_apply_kernel' -s 0 -c 1 -o "$OUT/k3" \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > "$OUT/ncu_k3.log" 2>&1
echo "k3 rc=$?"
