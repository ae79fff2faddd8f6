#!/usr/bin/env bash
# Re-entry check of HEAD: GPU suite, smoke, cfg3 + cfg1 bench lines.
set -u
TAG=${1:-r02h2}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > "$OUT/smi.txt" 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
tail -n 3 "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
tail -n 2 "$OUT/smoke.log"
for cfg in cfg3 cfg1; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 > "$OUT/bench_$cfg.json" 2> "$OUT/bench_$cfg.err"
  tail -c 600 "$OUT/bench_$cfg.json"; echo
done
