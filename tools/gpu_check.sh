#!/usr/bin/env bash
# One gpurun call: GPU parity tests, smoke, a short bench, the ncu launch list
# and one `ncu --set full` capture of the dominant kernel.
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tag]'
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > "$OUT/smi.txt" 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 400 python bench.py --steps 3 --warmup 3 > "$OUT/bench.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench.log"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > "$OUT/ncu_launch.log" 2>&1; echo "ncu launches rc=$?" >> "$OUT/ncu_launch.log"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_lse -s 2 -c 1 \
  -o "$OUT/tc_lse_full" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > "$OUT/ncu_full.log" 2>&1; echo "ncu full rc=$?" >> "$OUT/ncu_full.log"
for f in "$OUT"/*.log; do echo "== $f"; tail -n 3 "$f"; done
