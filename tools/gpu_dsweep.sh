#!/usr/bin/env bash
# N2 evidence: FMA vs tcgen05 half-step over d (timing + ncu pipe counters).
#   gpurun -- 'bash tools/gpu_dsweep.sh TAG'
set -u
TAG=${1:-dsweep}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python tools/dsweep.py > "$OUT/dsweep.jsonl" 2> "$OUT/dsweep.err"; echo "dsweep rc=$?"
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:"lse" --csv --log-file "$OUT/dsweep_ncu.csv" \
  python tools/dsweep.py --passes 1 --warm 0 > "$OUT/dsweep_ncu.log" 2>&1; echo "ncu rc=$?"
