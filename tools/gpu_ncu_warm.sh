#!/usr/bin/env bash
# ncu --set full of one warm-bound K1 pass (7th tq launch of the first cfg3 step)
# and of the screened cold pass (1st), with source mapping.
set -u
TAG=${1:-ncu_warm}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_lse_tq -s 6 -c 1 \
  -o "$OUT/k1_warm" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity \
  > "$OUT/ncu_warm.log" 2>&1; echo "warm rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_apply -c 1 \
  -o "$OUT/k3" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity \
  > "$OUT/ncu_k3.log" 2>&1; echo "k3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity \
  > "$OUT/ncu_launch.log" 2>&1; echo "launches rc=$?"
ls -la "$OUT"
