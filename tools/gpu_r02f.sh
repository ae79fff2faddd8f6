#!/usr/bin/env bash
set -u
TAG=${1:-r02f}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_multi_gpu_paths.py -x -q -s > "$OUT/multi.log" 2>&1; echo "multi rc=$?" >> "$OUT/multi.log"
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 1 > "$OUT/bench_cfg4.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench_cfg4.log"
timeout 600 python bench.py --config cfg5 --steps 2 --warmup 1 > "$OUT/bench_cfg5.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench_cfg5.log"
for f in "$OUT"/*.log; do echo "== $f"; tail -n 6 "$f" | cut -c1-1500; done
