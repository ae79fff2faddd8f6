#!/usr/bin/env bash
set -u
TAG=${1:-r02e}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python tools/plan_cache_diag.py > "$OUT/plan_diag.log" 2>&1; echo "diag rc=$?" >> "$OUT/plan_diag.log"
timeout 900 python -m pytest tests/test_tensor_gpu.py -x -q -s -k "persistent or graph or warm_start or warm_resolve or bit_identical" > "$OUT/new.log" 2>&1; echo "new rc=$?" >> "$OUT/new.log"
timeout 900 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 > "$OUT/bench_cfg1.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench_cfg1.log"
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 > "$OUT/bench_cfg2.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench_cfg2.log"
timeout 600 python tools/pass_profile.py --config cfg3 --reps 2 > "$OUT/pass_profile.log" 2>&1; echo "pp rc=$?" >> "$OUT/pass_profile.log"
for f in "$OUT"/*.log; do echo "== $f"; tail -n 6 "$f" | cut -c1-1200; done
