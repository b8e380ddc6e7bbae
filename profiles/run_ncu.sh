#!/bin/bash
# Profiling recipe used for profiles/ (run under gpurun on one B200).
# 1) launch list of one fwd+bwd step at the 7B shape (cold-cache, serialised:
#    compare kernel SHARES with bench.py's live per-kernel events, not absolutes)
# 2) one `--set full` capture of each tcgen05 kernel class of that step.
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
K='regex:state_scan_kernel|fwd_parallel_kernel|bwd_parallel_kernel|gates_|assemble_kernel|states_to_bf16'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k "$K" -s 30 -c 10 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k 'regex:state_scan_kernel|fwd_parallel_kernel|bwd_parallel_kernel' -s 18 -c 6 \
    -o $OUT/prof_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/prof_full.log 2>&1
ls -la $OUT
