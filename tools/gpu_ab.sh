#!/usr/bin/env bash
# A/B runs: tensor-path tests (per setting), then each config under each env setting.
#   bash tools/gpu_ab.sh TAG "cfg2 cfg3" "FSK_MINIT=0" "FSK_MINIT=1" ...
set -u
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
i=0
for setting in "$@"; do
  env $setting timeout 400 python -m pytest tests/test_tensor_gpu.py -x -q -s > "$OUT/pytest_$i.log" 2>&1; echo "rc=$? [$setting]" >> "$OUT/pytest_$i.log"
  for c in $CFGS; do
    env $setting timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > "$OUT/bench_${c}_$i.log" 2>&1
    echo "[$setting]" >> "$OUT/bench_${c}_$i.log"
  done
  i=$((i+1))
done
python - "$OUT" <<'PY'
import json, sys, glob
for f in sorted(glob.glob(sys.argv[1] + "/bench_*.log")):
    lines = open(f).read().splitlines()
    js = [l for l in lines if l.startswith("{")]
    if not js:
        print(f, "NO JSON", lines[-3:]); continue
    d = json.loads(js[-1])
    print(f.split("/")[-1], lines[-1], "value %.3f" % d["value"], "half %.2f grad %.2f" % (d.get("half_step_ms", 0), d.get("grad_ms", 0)),
          "e2e %.3f" % d["e2e"]["value"] if "e2e" in d else "", "live %s" % d.get("block_skipping", {}).get("live_fraction"))
PY
for f in "$OUT"/pytest_*.log; do echo "== $f"; grep -E "shard vs full|passed|failed|rc=" "$f" | sort | uniq -c | tail -n 6; done
