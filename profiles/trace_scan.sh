#!/bin/bash
# scan traces at the 7B shape (last eager launch of the bench): fwd L=128 (split), fwd L=256, bwd L=128
mkdir -p gpurun_out
a="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1"
TFLA_TRACE_SCAN=gpurun_out/scan_fwd_L128.txt TFLA_NO_FUSED_FWD=1 timeout 300 python bench.py $a > /dev/null 2>&1
TFLA_TRACE_SCAN=gpurun_out/scan_fwd_L256.txt timeout 300 python bench.py --L 256 $a > /dev/null 2>&1
TFLA_TRACE_SCAN=gpurun_out/scan_fwd_L256_sig.txt timeout 300 python bench.py --L 256 --variant sig $a > /dev/null 2>&1
TFLA_TRACE_SCAN=gpurun_out/scan_bwd_L128.txt TFLA_TRACE_SCAN_DIR=bwd timeout 300 python bench.py $a > /dev/null 2>&1
for f in scan_fwd_L128 scan_fwd_L256 scan_fwd_L256_sig scan_bwd_L128; do echo "== $f"; python profiles/trace_scan.py gpurun_out/$f.txt | grep -v "^  st"; done
