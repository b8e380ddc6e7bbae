#!/bin/bash
# backward scan at L=128 (no d_g): lazy staging wait; 64- vs 128-row stages
k() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items() if 'scan' in k})"; }
for E in X=1 TFLA_SCAN_R128=1; do
  echo "== $E long L=128"; timeout 300 env $E python bench.py --B 1 --NH 8 --S 65536 --L 128 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | k
  echo "== $E 7B L=128"; timeout 300 env $E python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | k
done
