#!/usr/bin/env bash
# ncu evidence for the current kernels: launch list of one cfg3 bench step and
# one `--set full` capture of each dominant kernel.   bash tools/gpu_profile.sh TAG
set -u
TAG=${1:-prof}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > "$OUT/ncu_launch.log" 2>&1; echo "launches rc=$?"
# screened K1 (the 3rd launch of the step is a steady-state f-update) and K3 of the gradient
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_lse_tq -s 4 -c 1 \
  -o "$OUT/k1" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > "$OUT/ncu_k1.log" 2>&1; echo "k1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_apply -c 1 \
  -o "$OUT/k3" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > "$OUT/ncu_k3.log" 2>&1; echo "k3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_lse_chunked -c 1 \
  -o "$OUT/k1c" python bench.py --config cfg4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > "$OUT/ncu_k1c.log" 2>&1; echo "k1c rc=$?"
ls -la "$OUT"
