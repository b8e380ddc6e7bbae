#!/bin/bash
# state-scan experiments at L=256 (7B shape): exp vs sig, 64- vs 128-column tiles
run() { echo "== $*"; timeout 300 env "$@" python bench.py --L 256 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items()})"; }
run X=1
run TFLA_SCAN_FWD_N=128 TFLA_SCAN_BWD_N=128

echo "== sig"; timeout 300 python bench.py --L 256 --variant sig --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k: v['ms'] for k, v in d['kernels'].items()})"
