#!/bin/bash
# other head shapes / batch layouts (mLSTMexp, L=128): tokens/s and tensor fraction
for cfg in "8 8 8192 256 512" "16 8 8192 256 512" "4 16 8192 256 512" "8 8 8192 128 256" "16 4 4096 128 256" "8 8 8192 128 512" "32 8 2048 256 512"; do
  set -- $cfg
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --B $1 --NH $2 --S $3 --dqk $4 --dhv $5 2>/dev/null | tail -1 | \
    python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('B=$1 NH=$2 S=$3 dqk=$4 dhv=$5: %.3f ms/step %.2f Mtok/s tensor_frac %.3f fwd %.3f ms | %s' % (d['ms_per_step'], d['value']/1e6, d['tensor_peak_frac'], d['fwd']['ms_per_step'], ' '.join('%s=%.3f'%(k,v['ms']) for k,v in d['kernels'].items())))"
done
