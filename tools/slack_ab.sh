#!/usr/bin/env bash
set -u
for sl in 8 2; do
  for rep in 1 2; do
    FSK_SCREEN_SLACK=$sl timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$sl', round(d['value'],3), round(d['half_step_mean_ms'],1), round(d['grad_ms'],1), round(d['block_skipping']['live_fraction'],4), d['clocks']['sm_mhz'])"
  done
done
FSK_SCREEN_SLACK=2 timeout 300 python -m pytest tests/test_tensor_gpu.py -x -q 2>&1 | tail -1
