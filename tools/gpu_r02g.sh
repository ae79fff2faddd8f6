#!/usr/bin/env bash
set -u
TAG=${1:-r02g}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_multi_gpu_paths.py -x -q -s > "$OUT/multi.log" 2>&1; echo "multi rc=$?" >> "$OUT/multi.log"
timeout 900 python bench.py --steps 5 --warmup 3 > "$OUT/bench_cfg3.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench_cfg3.log"
FSK_WARM=0 FSK_SCREEN=0 timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > "$OUT/bench_cfg3_dense.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench_cfg3_dense.log"
for f in "$OUT"/*.log; do echo "== $f"; tail -n 6 "$f" | cut -c1-1500; done
