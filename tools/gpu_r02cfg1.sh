#!/usr/bin/env bash
# cfg1 A/B: resident-cloud persistent solve vs the staging kernel, fused fp64 gradient
# vs the two-pass one; cfg1 launch list and a --set full capture of the persistent kernel.
#   gpurun -- 'bash tools/gpu_r02cfg1.sh TAG'
set -u
TAG=${1:-r02cfg1}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -q -k "persistent or small or cfg1 or golden or grad or parity" > "$OUT/pytest.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest.log"
tail -n 3 "$OUT/pytest.log"
for v in "1 1" "0 1" "1 0" "1 1"; do
  set -- $v
  FSK_SMALL_RESIDENT=$1 FSK_GRAD_FUSED=$2 timeout 300 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > "$OUT/bench_cfg1_$1$2.json" 2> "$OUT/bench_cfg1_$1$2.err"
  python -c "
import json
d=json.loads(open('$OUT/bench_cfg1_$1$2.json').read().strip().splitlines()[-1])
print('res=$1 fused=$2', d.get('value'), d.get('half_step_ms'), d.get('grad_ms'), (d.get('e2e') or {}).get('value'), (d.get('parity') or {}))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --config cfg1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity \
  > "$OUT/ncu_launch.log" 2>&1; echo "launches rc=$?" >> "$OUT/ncu_launch.log"
python tools/ncu_summary.py "$OUT/launches.csv" --launches | head -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_solve_res -c 1 -o "$OUT/small" \
  python bench.py --config cfg1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > "$OUT/ncu_small.log" 2>&1
echo "small rc=$?"
