#!/bin/bash
# ncu bundle for one chunk size (split path): launch list of one fwd+bwd step
# (cold, serialised) + --set full of the tcgen05 kernels of one step.
# usage: run_ncu_L.sh <L> <tag> [bench args]
L=$1; TAG=$2; shift 2
mkdir -p gpurun_out
K='regex:state_scan_kernel|fwd_parallel_kernel|fwd_fused_kernel|bwd_fused_kernel|bwd_parallel_kernel|gates_|mscan_kernel|assemble_kernel|qn_kernel|nscan_kernel'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k "$K" -s 40 -c 14 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --L $L --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 "$@" > gpurun_out/${TAG}_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k 'regex:state_scan_kernel|fwd_parallel_kernel|bwd_parallel_kernel|fwd_fused_kernel|bwd_fused_kernel' -s 6 -c 6 \
    -o gpurun_out/${TAG}_full -f python bench.py --L $L --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 "$@" > gpurun_out/${TAG}_full.log 2>&1
python profiles/ncu_top.py gpurun_out/${TAG}_full.ncu-rep 10 > gpurun_out/${TAG}_full.txt 2>&1
tail -3 gpurun_out/${TAG}_full.log
