#!/bin/bash
# fused backward: L2 prefetch of the next tile's q/k/dH/v rows, issued at group g (0 = off)
for g in 0 1 3 5 8; do
echo "== TFLA_BWDF_PREFETCH=$g"; timeout 300 env TFLA_BWDF_PREFETCH=$g python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items() if k.startswith('bwd')})"
done
