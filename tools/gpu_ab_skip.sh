#!/usr/bin/env bash
# A/B of the skip threshold T (default 26 + ceil(log2 m) vs the fixed 58) on cfg3 and
# cfg2, with the label and benchmark-config parity tests.
set -u
TAG=${1:-skip}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_tensor_gpu.py tests/test_bench_parity_gpu.py -q -x > "$OUT/pytest.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest.log"
for cfg in cfg3 cfg2; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_${cfg}_T.json" 2> "$OUT/bench_${cfg}_T.err"
  FSK_SKIP_LOG2=58 timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/bench_${cfg}_58.json" 2> "$OUT/bench_${cfg}_58.err"
done
timeout 600 python tools/pass_profile.py --config cfg3 --reps 1 > "$OUT/pass_profile.log" 2>&1
tail -n 3 "$OUT/pytest.log"
for f in "$OUT"/bench_*.json; do echo "== $f"; python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['half_step_mean_ms'], d.get('grad_ms'), d['roofline']['frac'], d.get('block_skipping',{}).get('live_fraction'), d.get('parity',{}).get('max_rel_err'), d.get('parity',{}).get('grad_max_rel_err'), d['clocks']['sm_mhz'])"; done
