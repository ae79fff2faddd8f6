#!/usr/bin/env bash
# Round-2 re-entry check: full GPU suite, smoke, every config's bench line,
# a dense cfg3 line and the reference arm.   gpurun -- 'bash tools/gpu_r02i.sh TAG'
set -u
TAG=${1:-r02i}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > "$OUT/smi.txt" 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
for cfg in cfg3 cfg2 cfg1 cfg4 cfg5; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 > "$OUT/bench_$cfg.json" 2> "$OUT/bench_$cfg.err"
  echo "$cfg rc=$?" >> "$OUT/bench_$cfg.err"
done
FSK_WARM=0 FSK_SCREEN=0 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parity > "$OUT/bench_cfg3_dense.json" 2> "$OUT/bench_cfg3_dense.err"
for f in "$OUT"/*.log; do echo "== $f"; tail -n 6 "$f" | cut -c1-1500; done
for f in "$OUT"/bench_*.json; do echo "== $f"; cut -c1-900 "$f"; done
