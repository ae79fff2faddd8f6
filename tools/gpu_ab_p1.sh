#!/usr/bin/env bash
set -u
OUT=gpurun_out/${1:-p1}; mkdir -p "$OUT"
for sp in 1 2 4; do
  FSK_P1_SPLITS=$sp FSK_TP_SPLITS=8 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > "$OUT/b$sp.json" 2>/dev/null
  python -c "
import json; d=json.loads(open('$OUT/b$sp.json').read().strip().splitlines()[-1]); print('p1 splits $sp', round(d['value'],3), round(d['half_step_mean_ms'],2), d['block_skipping']['live_fraction'])"
  FSK_P1_SPLITS=$sp FSK_TP_SPLITS=8 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:tc_lse_tq_kernel --log-file "$OUT/l$sp.csv" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1
done
