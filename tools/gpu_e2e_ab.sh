#!/usr/bin/env bash
# e2e variance probe: per-call wall time over many calls, pool reserve off / on
set -u
TAG=${1:-e2eab}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
FSK_TIMING=1 REPS=10 timeout 900 python tools/e2e_timing.py cfg3 > "$OUT/timing_noreserve.log" 2>&1
FSK_POOL_RESERVE_GB=24 FSK_TIMING=1 REPS=10 timeout 900 python tools/e2e_timing.py cfg3 > "$OUT/timing_reserve.log" 2>&1
REPS=10 timeout 900 python tools/e2e_timing.py cfg3 > "$OUT/notiming_noreserve.log" 2>&1
FSK_POOL_RESERVE_GB=24 REPS=10 timeout 900 python tools/e2e_timing.py cfg3 > "$OUT/notiming_reserve.log" 2>&1
for f in "$OUT"/*.log; do echo "== $f"; grep -E "^rep" $f | tr '\n' ' '; echo; done
grep -E "rep|iterations|gradient|upload|marginals" "$OUT/timing_reserve.log"
