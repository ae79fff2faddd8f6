#!/usr/bin/env bash
set -u
TAG=${1:-r02h}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_tensor_gpu.py -x -q > "$OUT/tensor.log" 2>&1; echo "tensor rc=$?" >> "$OUT/tensor.log"
timeout 900 python -m pytest tests/test_bench_parity_gpu.py -x -q -s -k "bench_step or dense_mode" > "$OUT/parity.log" 2>&1; echo "parity rc=$?" >> "$OUT/parity.log"
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > "$OUT/bench_cfg3.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench_cfg3.log"
timeout 600 python tools/pass_profile.py --config cfg3 --reps 2 > "$OUT/pass_profile.log" 2>&1; echo "pp rc=$?" >> "$OUT/pass_profile.log"
FSK_WARM=0 FSK_SCREEN=0 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parity > "$OUT/bench_cfg3_dense.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench_cfg3_dense.log"
for f in "$OUT"/*.log; do echo "== $f"; tail -n 5 "$f" | cut -c1-1200; done
