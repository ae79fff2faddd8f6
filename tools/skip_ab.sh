#!/usr/bin/env bash
# A/B of the skip threshold: the default library, then _build/libfsk_b200_skip58.so
# swapped in (run on a scratch copy of the repo, e.g. the gpurun box).
set -u
B=paper_2602_03067_b200/_build
cp $B/libfsk_b200.so /tmp/libfsk_b200_default.so
for lib in default skip58; do
  if [ $lib = skip58 ]; then cp $B/libfsk_b200_skip58.so $B/libfsk_b200.so; fi
  for rep in 1 2; do
    timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['value'],3), round(d['half_step_ms'],1), round(d['grad_ms'],1), round(d['block_skipping']['live_fraction'],4), d['clocks']['sm_mhz'])"
  done
  if [ $lib = skip58 ]; then timeout 300 python -m pytest tests/test_tensor_gpu.py -x -q 2>&1 | tail -1; fi
done
cp /tmp/libfsk_b200_default.so $B/libfsk_b200.so
