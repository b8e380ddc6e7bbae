#!/bin/bash
# per-kernel breakdown of the fwd+bwd step: 7B shape and long context, L = 128 / 256 / 512
k() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'fwd', round(d['fwd']['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items()})"; }
for L in 128 256 512; do
  echo "== long L=$L"; timeout 300 env "$@" python bench.py --B 1 --NH 8 --S 65536 --L $L --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | k
  echo "== 7B L=$L"; timeout 300 env "$@" python bench.py --L $L --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | k
done
