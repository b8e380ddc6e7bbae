#!/bin/bash
# Round-2 profile bundle (one gpurun call, 1 GPU):
#  1) the default bench line (headline, with cpu_baseline, e2e and the L sweep) -> gpurun_out/bench.json
#  2) ncu launch list of one full-batch fwd+bwd step at L=128 (--splits 1) and at L=256 -> *_launches.csv
#  3) ncu --set full of the tcgen05 kernels of one step at L=128 and L=256
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
K='regex:state_scan|fwd_parallel_kernel|fwd_fused_kernel|bwd_fused_kernel|bwd_parallel_kernel|gates_|mscan_kernel|assemble_kernel|qn_kernel|nscan_kernel'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k "$K" -s 24 -c 8 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 > gpurun_out/launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k 'regex:state_scan_kernel|fwd_fused_kernel|bwd_fused_kernel' -s 9 -c 3 \
    -o gpurun_out/prof_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 > gpurun_out/prof_full.log 2>&1
python profiles/ncu_top.py gpurun_out/prof_full.ncu-rep 12 > gpurun_out/prof_full.txt 2>&1
bash profiles/run_ncu_L.sh 256 L256
ls -la gpurun_out
