#!/bin/bash
# forward path comparison at the 7B shape, L=128: fused K12 vs split (K1 scan + wide K2), scan variants
run() { echo "== $*"; timeout 300 env "$@" python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'fwd', round(d['fwd']['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items()})"; }
run X=1
run TFLA_NO_FUSED_FWD=1
run TFLA_NO_FUSED_FWD=1 TFLA_SCAN2=1
