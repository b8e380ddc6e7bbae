#!/bin/bash
# split-backward barrier-wait traces (CTA 0) at L = 256 / 512
mkdir -p gpurun_out
for L in 256 512; do
TFLA_TRACE_BWDK=gpurun_out/bwdk_L$L timeout 300 python bench.py --L $L --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 > /dev/null 2>&1
for k in dq dk dv; do echo "L=$L $k: $(cat gpurun_out/bwdk_L${L}_$k.txt)"; done
done
