#!/usr/bin/env bash
# Screen-phase MMA grouping A/B (FSK_SCREEN_GROUP 1 / 2 / 4): cfg3 bench-step parity per
# setting (guarded), then cfg3 benches interleaved.   gpurun -- 'bash tools/gpu_ab_group.sh TAG'
set -u
TAG=${1:-r02group}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for g in 2 4; do
  FSK_SCREEN_GROUP=$g timeout 400 python -m pytest tests/test_bench_parity_gpu.py -x -q -k "cfg3" > "$OUT/pytest_cfg3_g$g.log" 2>&1
  rc=$?; echo "rc=$rc" >> "$OUT/pytest_cfg3_g$g.log"; tail -n 2 "$OUT/pytest_cfg3_g$g.log"
  [ $rc -eq 0 ] || exit 1
done
timeout 300 python -m pytest tests/test_tensor_gpu.py -x -q -k "ring" > "$OUT/pytest_ring.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_ring.log"; tail -n 2 "$OUT/pytest_ring.log"
i=0
for setting in 1 2 4 1 2 4; do
  FSK_SCREEN_GROUP=$setting timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > "$OUT/bench_cfg3_$i.log" 2>&1
  echo "[FSK_SCREEN_GROUP=$setting]" >> "$OUT/bench_cfg3_$i.log"
  i=$((i+1))
done
for g in 1 2 4; do
  FSK_SCREEN_GROUP=$g timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_lse_tq --csv --log-file "$OUT/l_$g.csv" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1
done
python - "$OUT" <<'PY'
import json, sys, glob, csv
for f in sorted(glob.glob(sys.argv[1] + "/bench_*.log")):
    lines = open(f).read().splitlines()
    js = [l for l in lines if l.startswith("{")]
    if not js:
        print(f, "NO JSON", lines[-3:]); continue
    d = json.loads(js[-1])
    print(f.split("/")[-1], lines[-1], "value %.3f" % d["value"], "half_mean %.2f" % d.get("half_step_mean_ms", 0),
          "frac %.3f" % d["roofline"]["frac"], "clk", d["clocks"]["sm_mhz"], "live %s" % d.get("block_skipping", {}).get("live_fraction"))
for f in sorted(glob.glob(sys.argv[1] + "/l_*.csv")):
    rows = [r for r in csv.reader(l for l in open(f) if not l.startswith("=="))]
    if not rows: continue
    h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value")
    big = [round(float(r[iv].replace(",", "")) / 1e6, 1) for r in rows[1:] if "1>" in r[ik][:40] and float(r[iv].replace(",", "")) > 5e7]
    print(f.split("/")[-1], "phase-1 launches (ms):", big)
PY
