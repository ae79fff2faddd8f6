#!/usr/bin/env bash
# Iteration run: targeted GPU tests, then the bench line, then (optionally) an
# ncu --set full capture of one kernel.   bash tools/gpu_iter.sh TAG [KERNEL_REGEX]
set -u
TAG=${1:-iter}
KREGEX=${2:-}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_tensor_gpu.py -x -q > "$OUT/pytest_tensor.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_tensor.log"
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 python bench.py --steps 3 --warmup 3 > "$OUT/bench.log" 2>&1; echo "rc=$?" >> "$OUT/bench.log"
if [ -n "$KREGEX" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -c 1 \
    -o "$OUT/full" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
    > "$OUT/ncu_full.log" 2>&1; echo "rc=$?" >> "$OUT/ncu_full.log"
fi
for f in "$OUT"/*.log; do echo "== $f"; tail -n 4 "$f" | cut -c1-600; done
