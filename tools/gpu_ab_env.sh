#!/usr/bin/env bash
# Generic A/B of one FSK_* switch: guarded bench-step parity and the tensor suite with the
# default build, then cfg3 / cfg2 benches interleaved over the settings (2 rounds) and the
# per-launch K1 times of one cfg3 step under each.
#   gpurun -- 'bash tools/gpu_ab_env.sh TAG FSK_HALF_LOAD "0 1"'
set -u
TAG=$1; VAR=$2; VALS=$3
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 400 python -m pytest tests/test_bench_parity_gpu.py -x -q -k "cfg3 or cfg2" > "$OUT/pytest_bench.log" 2>&1
rc=$?; echo "rc=$rc" >> "$OUT/pytest_bench.log"; tail -n 2 "$OUT/pytest_bench.log"
[ $rc -eq 0 ] || exit 1
timeout 900 python -m pytest tests/test_tensor_gpu.py -x -q > "$OUT/pytest_tensor.log" 2>&1
echo "rc=$?" >> "$OUT/pytest_tensor.log"; tail -n 2 "$OUT/pytest_tensor.log"
i=0
for rep in 1 2; do
for v in $VALS; do
  for c in cfg3 cfg2; do
    env $VAR=$v timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > "$OUT/bench_${c}_$i.log" 2>&1
    echo "[$VAR=$v]" >> "$OUT/bench_${c}_$i.log"
  done
  i=$((i+1))
done
done
for v in $VALS; do
  env $VAR=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:tc_lse_tq --csv --log-file "$OUT/l_$v.csv" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1
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
    h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value"); im = h.index("Metric Name")
    ts = [(r[ik][:40], float(r[iv].replace(",", "")) / 1e6) for r in rows[1:] if r[im] == "gpu__time_duration.sum"]
    p1 = [round(v, 1) for k, v in ts if "0, 1" in k and v > 50]
    warm = [v for k, v in ts if "0, 0" in k]
    print(f.split("/")[-1], "phase-1 ms", p1, "warm/phase-2: %d launches, total %.1f ms" % (len(warm), sum(warm)))
PY
