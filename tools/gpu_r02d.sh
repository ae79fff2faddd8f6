#!/usr/bin/env bash
set -u
TAG=${1:-r02d}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_tensor_gpu.py -x -q -s -k "persistent or graph or warm_start or warm_resolve or bit_identical" > "$OUT/new.log" 2>&1; echo "new rc=$?" >> "$OUT/new.log"
timeout 900 python -m pytest tests/test_bench_parity_gpu.py -x -q -s > "$OUT/parity.log" 2>&1; echo "parity rc=$?" >> "$OUT/parity.log"
timeout 900 python -m pytest tests -m gpu -q --deselect tests/test_bench_parity_gpu.py > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 > "$OUT/bench_cfg1.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench_cfg1.log"
bash tools/gpu_dsweep.sh $TAG
for f in "$OUT"/*.log; do echo "== $f"; tail -n 4 "$f" | cut -c1-1500; done
cat "$OUT/dsweep.jsonl"
