#!/usr/bin/env bash
set -u
OUT=gpurun_out/${1:-r02ab}; mkdir -p "$OUT"
timeout 1200 python -m pytest tests/test_tensor_gpu.py tests/test_bench_parity_gpu.py tests/test_parity_gpu.py tests/test_spec_acceptance_gpu.py tests/test_multi_gpu_paths.py -q -x > "$OUT/pytest.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest.log"
tail -n 3 "$OUT/pytest.log"
for cfg in cfg4 cfg5 cfg3; do
timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/$cfg.json" 2>/dev/null
python -c "
import json; d=json.loads(open('$OUT/$cfg.json').read().strip().splitlines()[-1]); print('$cfg', round(d['value'],3), d.get('half_step_mean_ms'), d.get('hvp_ms'), d.get('grad_ms'), round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],3), d.get('parity',{}).get('ok'))"
done
FSK_TIMING=1 timeout 600 python tools/hvp_timing.py cfg4 2>&1 | grep -E "hvp|rep" | tail -8
