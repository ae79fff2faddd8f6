#!/usr/bin/env bash
# Round-2 GPU check: benchmark-config parity tests (verbose), the full GPU suite,
# a cfg3 bench line with the parity field, and a dense (no skipping) cfg3 line.
#   gpurun --timeout 3000 -- 'bash tools/gpu_r02.sh TAG'
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > "$OUT/smi.txt" 2>&1
timeout 900 python -m pytest tests/test_bench_parity_gpu.py -x -q -s > "$OUT/parity.log" 2>&1; echo "parity rc=$?" >> "$OUT/parity.log"
timeout 900 python -m pytest tests -m gpu -q --deselect tests/test_bench_parity_gpu.py > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 600 python bench.py --steps 5 --warmup 3 > "$OUT/bench.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench.log"
for f in "$OUT"/*.log; do echo "== $f"; tail -n 4 "$f" | cut -c1-3000; done
