#!/usr/bin/env bash
# current-state numbers: every config's bench line, dense cfg3, cfg2 pass profile
set -u
TAG=${1:-r02w}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for cfg in cfg3 cfg2 cfg1 cfg4 cfg5; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 > "$OUT/bench_$cfg.json" 2> "$OUT/bench_$cfg.err"
done
FSK_WARM=0 FSK_SCREEN=0 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parity > "$OUT/bench_cfg3_dense.json" 2> "$OUT/bench_cfg3_dense.err"
FSK_DEBUG_PASS=1 timeout 300 python tools/pass_profile.py --config cfg2 --reps 2 > "$OUT/pass_profile_cfg2.log" 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
for f in "$OUT"/bench_*.json; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','half_step_mean_ms','grad_ms','hvp_ms')}, 'frac', (d.get('roofline') or {}).get('frac'), 'e2e', (d.get('e2e') or {}).get('value'), 'clk', (d.get('clocks') or {}).get('sm_mhz'), 'parity', (d.get('parity') or {}).get('ok'))" 2>&1 | tail -1; done
tail -n 25 "$OUT/pass_profile_cfg2.log"
