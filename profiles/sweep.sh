#!/bin/bash
# chunk-size sweep (BASELINE config 3 / 7B shape): one bench line per (variant, L)
for v in ${VARIANTS:-exp sig}; do
  for L in ${LS:-64 128 256 512 1024}; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --variant $v --L $L "$@" 2>/dev/null | tail -1 | \
      python -c "
import json,sys; d=json.loads(sys.stdin.read())
ks=' '.join('%s=%.3f'%(k,v['ms']) for k,v in d['kernels'].items())
print('$v L=$L ms/step %.3f Mtok/s %.2f tensor_frac %.3f | %s' % (d['ms_per_step'], d['value']/1e6, d['tensor_peak_frac'], ks))"
  done
done
