#!/bin/bash
# scan traces at the 7B shape: bwd L=128 (headline) and L=512, fwd L=256
mkdir -p gpurun_out
a="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1"
TFLA_TRACE_SCAN=gpurun_out/scan_bwd_L128.txt TFLA_TRACE_SCAN_DIR=bwd timeout 300 python bench.py $a > /dev/null 2>&1
TFLA_TRACE_SCAN=gpurun_out/scan_bwd_L512.txt TFLA_TRACE_SCAN_DIR=bwd timeout 300 python bench.py --L 512 $a > /dev/null 2>&1
TFLA_TRACE_SCAN=gpurun_out/scan_fwd_L256.txt timeout 300 python bench.py --L 256 $a > /dev/null 2>&1
for f in scan_bwd_L128 scan_bwd_L512 scan_fwd_L256; do echo "== $f"; python profiles/trace_scan.py gpurun_out/$f.txt; done
