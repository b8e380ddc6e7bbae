#!/bin/bash
# --set full of the headline (L=128) step's kernels: fwd_fused, bwd_fused, state_scan (bwd)
TAG=${1:-r02h}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k 'regex:state_scan_kernel|fwd_fused_kernel|bwd_fused_kernel' -s 3 -c 3 \
    -o gpurun_out/${TAG}_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 > gpurun_out/${TAG}_full.log 2>&1
python profiles/ncu_top.py gpurun_out/${TAG}_full.ncu-rep 10 > gpurun_out/${TAG}_full.txt 2>&1
tail -3 gpurun_out/${TAG}_full.log
