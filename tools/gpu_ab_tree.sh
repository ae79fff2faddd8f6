#!/usr/bin/env bash
# Same-box A/B of two builds: the tree at .abold (a git worktree of an earlier commit,
# built in place) and the working tree, interleaved: cfg3, cfg2 and dense cfg3 lines.
# Optional: EXTRA="VAR=value" adds a third arm, the working tree under that setting.
#   gpurun -- 'EXTRA=FSK_HALF_LOAD=0 bash tools/gpu_ab_tree.sh TAG'
set -u
TAG=${1:-r02tree}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_bench_parity_gpu.py tests/test_tensor_gpu.py -x -q > "$OUT/pytest.log" 2>&1
rc=$?; echo "rc=$rc" >> "$OUT/pytest.log"; tail -n 2 "$OUT/pytest.log"
[ $rc -eq 0 ] || exit 1
for r in 1 2; do
  for t in old new ${EXTRA:+extra}; do
    if [ $t = old ]; then d=.abold; else d=.; fi
    if [ $t = extra ]; then e="$EXTRA"; else e="FSK_NONE=1"; fi
    (cd $d && env $e timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity) > "$OUT/c3_${t}_$r.json" 2>/dev/null
    (cd $d && env $e timeout 300 python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-parity) > "$OUT/c2_${t}_$r.json" 2>/dev/null
    (cd $d && env $e FSK_WARM=0 FSK_SCREEN=0 timeout 400 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parity) > "$OUT/d3_${t}_$r.json" 2>/dev/null
  done
done
for f in "$OUT"/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['value'],3), 'half_mean', round(d['half_step_mean_ms'],3), 'clk', d['clocks']['sm_mhz'])"; done
