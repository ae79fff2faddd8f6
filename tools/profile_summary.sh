#!/usr/bin/env bash
# Markdown summary of a tools/gpu_r02final.sh capture directory (bench lines, launch list,
# full captures) for profiles/.   bash tools/profile_summary.sh gpurun_out/TAG "title" > profiles/X.md
set -u
O=$1; TITLE=$2
echo "# $TITLE"; echo
echo "Source: \`tools/gpu_r02final.sh\` → \`$O\` ($(grep -o '[0-9]* passed' $O/pytest_gpu.log | tail -1) in \`pytest -m gpu\`, $(tail -n 2 $O/smoke.log | head -1 | cut -c1-40)). Bench lines: 3 timed steps, 3 warm-up."; echo
echo "| config | value (it/s) | e2e (it/s, C ABI, host buffers) | roofline frac | parity | SM MHz |"
echo "|---|---|---|---|---|---|"
for c in cfg1 cfg2 cfg3 cfg3_dense cfg4 cfg5; do python - $O/bench_$c.json $c <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
e=(d.get('e2e') or {}).get('value'); r=(d.get('roofline') or {}).get('frac'); p=(d.get('parity') or {}).get('ok')
print(f"| {sys.argv[2]} | {d['value']:.4g} | {'%.4g'%e if e else '-'} | {'%.3f'%r if r else '-'} | {p if p is not None else '-'} | {(d.get('clocks') or {}).get('sm_mhz')} |")
PY
done
python - $O/bench_reference.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); c=d['cpu_baseline']
print(f"| reference arm (cfg3, oracle/_ref, {c['cores']} host cores) | {d['value']:.3g} | - | - | - | - |")
PY
echo
python tools/ncu_summary.py $O/launches.csv --launches
echo; echo "### cfg3 warm-bound K1 (9th launch of a step)"; python tools/ncu_summary.py $O/k1_warm.ncu-rep
echo; echo "### cfg3 screen phase 1 (first cold pass)"; python tools/ncu_summary.py $O/k1_screen.ncu-rep
echo; echo "### cfg3 K3 (gradient transport)"; python tools/ncu_summary.py $O/k3.ncu-rep
echo; echo "### cfg4 chunked warm K1 (d = 1024)"; python tools/ncu_summary.py $O/k1c_warm.ncu-rep
