#!/bin/bash
# long context (BASELINE configs[3]: B=1 NH=8 S=65536) at L = 128 / 256 / 512
for L in 128 256 512; do
echo "== L=$L"; timeout 300 python bench.py --B 1 --NH 8 --S 65536 --L $L --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items()})"
done
