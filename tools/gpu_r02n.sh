#!/usr/bin/env bash
# half-granular live sets: tests first (short timeouts), then cfg3/cfg2 benches + pass profile
set -u
TAG=${1:-r02m}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 300 python -m pytest tests/test_tensor_gpu.py -q -x -k "warm or screen or half_step_parity" > "$OUT/pytest_quick.log" 2>&1; echo "quick rc=$?" >> "$OUT/pytest_quick.log"
tail -n 4 "$OUT/pytest_quick.log"
grep -q "quick rc=0" "$OUT/pytest_quick.log" || exit 1
timeout 900 python -m pytest tests/test_tensor_gpu.py tests/test_bench_parity_gpu.py -q -x > "$OUT/pytest.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest.log"
tail -n 4 "$OUT/pytest.log"
for cfg in cfg3 cfg2; do
timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_$cfg.json" 2> "$OUT/bench_$cfg.err"
python -c "
import json; d=json.loads(open('$OUT/bench_$cfg.json').read().strip().splitlines()[-1]); print('$cfg', d['value'], d['half_step_mean_ms'], d.get('grad_ms'), d['roofline']['frac'], d.get('block_skipping',{}).get('live_fraction'), d.get('parity',{}).get('max_rel_err'), d.get('parity',{}).get('grad_max_rel_err'), d['clocks']['sm_mhz'], d['e2e']['value'])"
done
FSK_DEBUG_PASS=1 timeout 600 python tools/pass_profile.py --config cfg3 --reps 2 > "$OUT/pass_profile.log" 2>&1
grep -v "fsk pass" "$OUT/pass_profile.log" | tail -22; grep "fsk pass" "$OUT/pass_profile.log" | head -8
