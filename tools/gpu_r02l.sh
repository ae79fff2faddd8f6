#!/usr/bin/env bash
# two-phase cold pass: tests, cfg3 bench, pass profile, launch list, ncu of phase 1.
set -u
TAG=${1:-r02l}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_tensor_gpu.py tests/test_bench_parity_gpu.py -q -x > "$OUT/pytest.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest.log"
tail -n 3 "$OUT/pytest.log"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_cfg3.json" 2> "$OUT/bench_cfg3.err"
timeout 600 python tools/pass_profile.py --config cfg3 --reps 1 > "$OUT/pass_profile.log" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity \
  > "$OUT/ncu_launch.log" 2>&1; echo "launches rc=$?" >> "$OUT/ncu_launch.log"
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_lse_tq_kernelILb0ELb1E' -s 0 -c 1 -o "$OUT/k1_screen" \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > "$OUT/ncu_screen.log" 2>&1
echo "screen rc=$?" >> "$OUT/ncu_screen.log"
python -c "
import json; d=json.loads(open('$OUT/bench_cfg3.json').read().strip().splitlines()[-1]); print(d['value'], d['half_step_mean_ms'], d.get('grad_ms'), d['roofline']['frac'], d.get('block_skipping',{}).get('live_fraction'), d.get('parity'), d['clocks']['sm_mhz'], d['e2e'])"
head -12 "$OUT/pass_profile.log"
