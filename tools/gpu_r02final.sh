#!/usr/bin/env bash
# Round-2 evidence: full GPU suite, smoke, every config's bench line (+ dense cfg3, reference
# arm), cfg3 ncu launch list with DRAM and --set full captures of warm K1 / screen phase 1 / K3,
# cfg4 chunked warm K1 capture.   gpurun -- 'bash tools/gpu_r02final.sh TAG'
set -u
TAG=${1:-r02final}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > "$OUT/smi.txt" 2>&1
timeout 1500 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
tail -n 3 "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
tail -n 2 "$OUT/smoke.log"
for cfg in cfg3 cfg2 cfg1 cfg4 cfg5; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 > "$OUT/bench_$cfg.json" 2> "$OUT/bench_$cfg.err"
done
FSK_WARM=0 FSK_SCREEN=0 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parity > "$OUT/bench_cfg3_dense.json" 2> "$OUT/bench_cfg3_dense.err"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
for f in "$OUT"/bench_*.json; do echo "== $f"; python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','half_step_mean_ms','grad_ms','hvp_ms')}, 'frac', (d.get('roofline') or {}).get('frac'), 'e2e', (d.get('e2e') or {}).get('value'), 'clk', (d.get('clocks') or {}).get('sm_mhz'), 'parity', (d.get('parity') or {}).get('ok'))" 2>&1 | tail -1; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity \
  > "$OUT/ncu_launch.log" 2>&1; echo "launches rc=$?" >> "$OUT/ncu_launch.log"
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_lse_tq_kernelILb0ELb0E' -s 8 -c 1 -o "$OUT/k1_warm" \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > "$OUT/ncu_warm.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_lse_tq_kernelILb0ELb1E' -s 0 -c 1 -o "$OUT/k1_screen" \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > "$OUT/ncu_screen.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_apply_kernel -c 1 \
  -o "$OUT/k3" python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > "$OUT/ncu_k3.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k 'regex:tc_lse_chunked_kernelILb0E' -s 10 -c 1 -o "$OUT/k1c_warm" \
  python bench.py --config cfg4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-parity > "$OUT/ncu_k1c.log" 2>&1
ls -la "$OUT"
