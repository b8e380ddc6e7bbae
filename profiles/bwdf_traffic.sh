#!/bin/bash
# fused backward: time (bench) + DRAM bytes of one launch (ncu)
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items()})"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum --clock-control none -k regex:bwd_fused_kernel -s 2 -c 1 --csv --log-file /tmp/bwdf_ncu.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 > /dev/null 2>&1
grep -v "^==" /tmp/bwdf_ncu.csv | python -c "
import csv,sys
for r in csv.DictReader(sys.stdin):
    print(r['Metric Name'], r['Metric Value'], r['Metric Unit'])"
