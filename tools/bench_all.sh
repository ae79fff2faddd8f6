#!/usr/bin/env bash
# Every BASELINE config through bench.py (one JSON line each) + the reference arm.
#   bash tools/bench_all.sh TAG
set -u
TAG=${1:-bench}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for cfg in cfg3 cfg2 cfg1 cfg4 cfg5; do
  timeout 500 python bench.py --config $cfg --steps 3 --warmup 3 > "$OUT/bench_$cfg.json" 2> "$OUT/bench_$cfg.err"
  echo "$cfg rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_reference_cfg3.json" 2> "$OUT/bench_reference.err"
echo "reference rc=$?"
for f in "$OUT"/bench_*.json; do echo "== $f"; cut -c1-400 "$f"; done
