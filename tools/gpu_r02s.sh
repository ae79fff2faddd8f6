#!/usr/bin/env bash
# e2e phase breakdown (cfg2, cfg3) + round-2 ncu evidence of the current cfg3 kernels
set -u
TAG=${1:-r02s}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for cfg in cfg2 cfg3; do FSK_TIMING=1 timeout 300 python tools/e2e_timing.py $cfg > "$OUT/e2e_$cfg.log" 2>&1; done
tail -n 30 "$OUT/e2e_cfg2.log"; tail -n 30 "$OUT/e2e_cfg3.log"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity \
  > "$OUT/ncu_launch.log" 2>&1; echo "launches rc=$?" >> "$OUT/ncu_launch.log"
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_lse_tq_kernelILb0ELb0E' -s 8 -c 1 -o "$OUT/k1_warm" \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > "$OUT/ncu_warm.log" 2>&1
echo "warm rc=$?" >> "$OUT/ncu_warm.log"
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_lse_tq_kernelILb0ELb1E' -s 0 -c 1 -o "$OUT/k1_screen" \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > "$OUT/ncu_screen.log" 2>&1
echo "screen rc=$?" >> "$OUT/ncu_screen.log"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_apply_kernel -c 1 \
  -o "$OUT/k3" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity \
  > "$OUT/ncu_k3.log" 2>&1; echo "k3 rc=$?" >> "$OUT/ncu_k3.log"
ls -la "$OUT"
