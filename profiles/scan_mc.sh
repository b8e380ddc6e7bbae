#!/bin/bash
# state scan: A (K / Q rows) multicast across the x-tile cluster (TFLA_SCAN_MC=1) vs one load per CTA
k() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items() if 'scan' in k or k in ('K1','K3')})"; }
for mc in 0 1; do
  E="TFLA_SCAN_MC=$mc"; [ $mc = 0 ] && E="X=1"
  echo "== $E long L=128"; timeout 300 env $E python bench.py --B 1 --NH 8 --S 65536 --L 128 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | k
  echo "== $E 7B L=128"; timeout 300 env $E python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | k
  echo "== $E 7B L=256"; timeout 300 env $E python bench.py --L 256 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | k
done
