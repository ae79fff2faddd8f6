#!/usr/bin/env bash
# device-decided passes: tests, 3 cfg3 bench runs (variance), cfg2, pass profile
set -u
TAG=${1:-r02x}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 300 python -m pytest tests/test_tensor_gpu.py -q -x -k "warm or screen or half_step_parity or history or run_to_run" > "$OUT/pytest_quick.log" 2>&1; echo "quick rc=$?" >> "$OUT/pytest_quick.log"
tail -n 3 "$OUT/pytest_quick.log"
grep -q "quick rc=0" "$OUT/pytest_quick.log" || exit 1
timeout 900 python -m pytest tests/test_tensor_gpu.py tests/test_bench_parity_gpu.py tests/test_multi_gpu_paths.py -q -x > "$OUT/pytest.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest.log"
tail -n 3 "$OUT/pytest.log"
for i in 1 2 3; do
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity > "$OUT/b$i.json" 2>/dev/null
python -c "
import json; d=json.loads(open('$OUT/b$i.json').read().strip().splitlines()[-1]); print('cfg3', $i, round(d['value'],3), round(d['half_step_ms'],2), round(d['half_step_mean_ms'],2), round(d['grad_ms'],1), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],3))"
done
timeout 300 python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline --no-parity > "$OUT/cfg2.json" 2>/dev/null
python -c "
import json; d=json.loads(open('$OUT/cfg2.json').read().strip().splitlines()[-1]); print('cfg2', round(d['value'],3), round(d['half_step_mean_ms'],3), d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value'],3))"
timeout 300 python tools/pass_profile.py --config cfg3 --reps 2 > "$OUT/pass_profile.log" 2>&1
tail -n 22 "$OUT/pass_profile.log"
