#!/usr/bin/env bash
# Lean MMA-chain issue A/B (FSK_LEAN_ISSUE 0: per-MMA elect and descriptor packing, 1: one
# elect per chain): guarded parity first, then interleaved benches and phase-1 launch times.
set -u
TAG=${1:-r02lean}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
FSK_LEAN_ISSUE=1 timeout 400 python -m pytest tests/test_bench_parity_gpu.py -x -q -k "cfg3 or cfg2" > "$OUT/pytest_bench.log" 2>&1
rc=$?; echo "rc=$rc" >> "$OUT/pytest_bench.log"; tail -n 2 "$OUT/pytest_bench.log"
[ $rc -eq 0 ] || exit 1
FSK_LEAN_ISSUE=1 timeout 900 python -m pytest tests/test_tensor_gpu.py -x -q > "$OUT/pytest_tensor.log" 2>&1
echo "rc=$?" >> "$OUT/pytest_tensor.log"; tail -n 2 "$OUT/pytest_tensor.log"
i=0
for rep in 1 2; do
for setting in "FSK_LEAN_ISSUE=0" "FSK_LEAN_ISSUE=1"; do
  env $setting timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > "$OUT/bench_cfg3_$i.log" 2>&1
  echo "[$setting]" >> "$OUT/bench_cfg3_$i.log"
  env $setting timeout 300 python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > "$OUT/bench_cfg2_$i.log" 2>&1
  echo "[$setting]" >> "$OUT/bench_cfg2_$i.log"
  i=$((i+1))
done
done
j=0
for setting in "FSK_LEAN_ISSUE=0" "FSK_LEAN_ISSUE=1"; do
  env $setting timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_lse_tq --csv --log-file "$OUT/l_$j.csv" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1
  echo "$setting" > "$OUT/l_$j.txt"; j=$((j+1))
done
python - "$OUT" <<'PY'
import json, sys, glob, csv
for f in sorted(glob.glob(sys.argv[1] + "/bench_*.log")):
    lines = open(f).read().splitlines()
    js = [l for l in lines if l.startswith("{")]
    if not js:
        print(f, "NO JSON", lines[-3:]); continue
    d = json.loads(js[-1])
    print(f.split("/")[-1], lines[-1], "value %.3f" % d["value"], "half_mean %.3f" % d.get("half_step_mean_ms", 0),
          "frac %.3f" % d["roofline"]["frac"], "clk", d["clocks"]["sm_mhz"])
for f in sorted(glob.glob(sys.argv[1] + "/l_*.csv")):
    rows = [r for r in csv.reader(l for l in open(f) if not l.startswith("=="))]
    if not rows: continue
    h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value")
    ts = [(r[ik][:40], float(r[iv].replace(",", "")) / 1e6) for r in rows[1:]]
    p1 = [round(v, 1) for k, v in ts if "0, 1" in k and v > 50]
    warm = [v for k, v in ts if "0, 0" in k]
    print(open(f[:-4] + ".txt").read().strip(), "phase-1 ms", p1, "warm/phase-2 total ms %.1f" % sum(warm))
PY
