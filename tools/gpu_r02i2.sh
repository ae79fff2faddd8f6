#!/usr/bin/env bash
# host-link check: new tests, e2e timing breakdown, cfg3 / cfg2 bench lines
set -u
TAG=${1:-r02i2}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_host_link_gpu.py tests/test_tensor_gpu.py tests/test_bench_parity_gpu.py tests/test_parity_gpu.py tests/test_spec_acceptance_gpu.py -m gpu -q -x > "$OUT/pytest.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest.log"
tail -n 15 "$OUT/pytest.log"
python tools/link_bw.py > "$OUT/link_bw.txt" 2>&1; cat "$OUT/link_bw.txt"
FSK_TIMING=1 REPS=3 timeout 600 python tools/e2e_timing.py cfg3 > "$OUT/timing_cfg3.log" 2>&1
tail -n 14 "$OUT/timing_cfg3.log"
for cfg in cfg3 cfg2 cfg1; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 > "$OUT/bench_$cfg.json" 2> "$OUT/bench_$cfg.err"
  python -c "
import json
d=json.loads(open('$OUT/bench_$cfg.json').read().strip().splitlines()[-1])
print('$cfg', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"
done
