#!/bin/bash
# scan traces at long context (B=1 NH=8 S=65536 L=128): deep (8-stage) vs 2-CTA/SM ring
mkdir -p gpurun_out
a="--B 1 --S 65536 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1"
TFLA_TRACE_SCAN=gpurun_out/scan_fwd_long_deep.txt timeout 300 python bench.py $a > /dev/null 2>&1
TFLA_TRACE_SCAN=gpurun_out/scan_fwd_long_2.txt TFLA_NO_DEEP_SCAN=1 timeout 300 python bench.py $a > /dev/null 2>&1
TFLA_TRACE_SCAN=gpurun_out/scan_bwd_long_deep.txt TFLA_TRACE_SCAN_DIR=bwd timeout 300 python bench.py $a > /dev/null 2>&1
for f in scan_fwd_long_deep scan_fwd_long_2 scan_bwd_long_deep; do echo "== $f"; python profiles/trace_scan.py gpurun_out/$f.txt | grep -v "^  "; done
