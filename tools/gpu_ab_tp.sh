#!/usr/bin/env bash
set -u
OUT=gpurun_out/${1:-tp}; mkdir -p "$OUT"
run() { # tag env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-parity > "$OUT/$tag.json" 2>/dev/null
  python -c "
import json; d=json.loads(open('$OUT/$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), round(d['half_step_mean_ms'],3), 'e2e', round(d['e2e']['value'],1))"
}
run tp1_dd FSK_TP_SPLITS=1
run tp4_dd FSK_TP_SPLITS=4
run tp4_host FSK_TP_SPLITS=4 FSK_DEVICE_DECIDE=0
run tp1_host FSK_TP_SPLITS=1 FSK_DEVICE_DECIDE=0
REPS=4 FSK_TIMING=1 timeout 300 python tools/e2e_timing.py cfg3 2>&1 | grep -E "rep|gradient"
for i in 1 2 3; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > "$OUT/c3_$i.json" 2>/dev/null; python -c "
import json; d=json.loads(open('$OUT/c3_$i.json').read().strip().splitlines()[-1]); print('cfg3', round(d['value'],3), 'e2e', round(d['e2e']['value'],3))"; done
