#!/bin/bash
# headline (7B shape, L=128) schedule / path variants
run() { echo "== $*"; timeout 300 env $1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sweep ${@:2} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items()})"; }
run X=1
run X=1 --splits 1
run X=1 --splits 4
run TFLA_NO_FUSED_BWD=1 --splits 1
