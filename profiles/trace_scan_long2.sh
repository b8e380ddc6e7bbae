#!/bin/bash
# backward scan traces at the default schedule: long context (deep ring) and the 7B shape (2 CTAs/SM), L=128
mkdir -p gpurun_out
a="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep"
TFLA_TRACE_SCAN=gpurun_out/scan_bwd_long_def.txt TFLA_TRACE_SCAN_DIR=bwd timeout 300 python bench.py --B 1 --S 65536 $a > /dev/null 2>&1
TFLA_TRACE_SCAN=gpurun_out/scan_bwd_7b_def.txt TFLA_TRACE_SCAN_DIR=bwd timeout 300 python bench.py $a > /dev/null 2>&1
TFLA_TRACE_SCAN=gpurun_out/scan_fwd_long_def.txt timeout 300 python bench.py --B 1 --S 65536 $a > /dev/null 2>&1
for f in scan_bwd_long_def scan_bwd_7b_def scan_fwd_long_def; do echo "== $f"; python profiles/trace_scan.py gpurun_out/$f.txt; done
