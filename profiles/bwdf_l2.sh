#!/bin/bash
# fused backward L2 last-use hints (TFLA_BWDF_L2 bits): bench kernel time + DRAM bytes per launch
for m in ${MODES:-0 1 2 4 8 15}; do
  echo "== TFLA_BWDF_L2=$m"
  TFLA_BWDF_L2=$m timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step', round(d['ms_per_step'],3), 'bwd_fused', d['kernels']['bwd_fused']['ms'])"
  TFLA_BWDF_L2=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bwd_fused_kernel -s 2 -c 1 --csv --log-file /tmp/bwdf_ncu.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 > /dev/null 2>&1
  grep -v "^==" /tmp/bwdf_ncu.csv | python -c "
import csv,sys
print('  ', {r['Metric Name']: r['Metric Value'] + ' ' + r['Metric Unit'] for r in csv.DictReader(sys.stdin)})"
done
