#!/usr/bin/env bash
# e2e phase breakdown (FSK_TIMING=1 marks synchronize the stream; numbers are per phase)
set -u
TAG=${1:-e2e}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for cfg in cfg3 cfg2; do
  FSK_TIMING=1 REPS=3 timeout 600 python tools/e2e_timing.py $cfg > "$OUT/timing_$cfg.log" 2>&1
  REPS=4 timeout 600 python tools/e2e_timing.py $cfg > "$OUT/notiming_$cfg.log" 2>&1
done
tail -n 40 "$OUT"/timing_cfg3.log "$OUT"/notiming_cfg3.log "$OUT"/timing_cfg2.log "$OUT"/notiming_cfg2.log
