#!/usr/bin/env bash
# GPU suite + ncu evidence of the cfg3 kernels (launch list; --set full of a warm
# K1 pass, the first screened K1 pass and K3).   gpurun -- 'bash tools/gpu_r02j.sh TAG'
set -u
TAG=${1:-r02j}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1500 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity \
  > "$OUT/ncu_launch.log" 2>&1; echo "launches rc=$?" >> "$OUT/ncu_launch.log"
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_lse_tq_kernelILb0ELb0E' -s 6 -c 1 -o "$OUT/k1_warm" \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > "$OUT/ncu_warm.log" 2>&1
echo "warm rc=$?" >> "$OUT/ncu_warm.log"
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_lse_tq_kernelILb0ELb1E' -s 0 -c 1 -o "$OUT/k1_screen" \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > "$OUT/ncu_screen.log" 2>&1
echo "screen rc=$?" >> "$OUT/ncu_screen.log"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_apply_kernel -c 1 \
  -o "$OUT/k3" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity \
  > "$OUT/ncu_k3.log" 2>&1; echo "k3 rc=$?" >> "$OUT/ncu_k3.log"
timeout 600 python tools/pass_profile.py --config cfg3 --reps 2 > "$OUT/pass_profile.log" 2>&1; echo "pp rc=$?" >> "$OUT/pass_profile.log"
for f in "$OUT"/*.log; do echo "== $f"; tail -n 5 "$f" | cut -c1-1500; done
ls -la "$OUT"
