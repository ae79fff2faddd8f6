for mb in 40 20 64 96; do
  for rep in 1 2; do
    FSK_WARM_RANGE_MB=$mb timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$mb', round(d['value'],3), round(d['half_step_ms'],1), round(d['grad_ms'],1), d['clocks']['sm_mhz'])"
  done
done
