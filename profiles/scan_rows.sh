#!/bin/bash
# state scan: 128-row stages (default where L % 128 == 0) vs 64-row stages (TFLA_SCAN_R64=1)
k() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items() if 'scan' in k})"; }
for E in TFLA_SCAN_R64=1 X=1; do
  echo "== $E long L=128"; timeout 300 env $E python bench.py --B 1 --NH 8 --S 65536 --L 128 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | k
  echo "== $E long L=256"; timeout 300 env $E python bench.py --B 1 --NH 8 --S 65536 --L 256 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | k
  echo "== $E 7B L=256"; timeout 300 env $E python bench.py --L 256 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | k
done
