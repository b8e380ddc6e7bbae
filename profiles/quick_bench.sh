#!/bin/bash
# quick perf check: parity suite + a short bench with per-kernel times
T=$(timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout=300 -x 2>&1 | tail -1)
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('ms/step %.3f  Mtok/s %.2f  tensor_frac %.3f' % (d['ms_per_step'], d['value']/1e6, d['tensor_peak_frac']))
for k,v in d['kernels'].items(): print('  %-16s %s' % (k, v))"
echo "TESTS: $T"
