#!/bin/bash
# BASELINE configs[3]: long context (B=1, NH=8, S=65536), chunk-size sweep:
# state memory (NC+1) x dqk x dhv per head vs step time
for v in exp sig; do
for L in 64 128 256 512 1024; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --B 1 --S 65536 --variant $v --L $L 2>/dev/null | tail -1 | \
    python -c "
import json,sys; d=json.loads(sys.stdin.read())
L=$L; NC=65536//L
st_f32=(NC+1)*256*512*4/2**20; st_bf16=NC*256*512*2/2**20
ks=' '.join('%s=%.3f'%(k,v['ms']) for k,v in d['kernels'].items())
print('$v L=%d NC=%d states/head fp32 %.0f MiB bf16 %.0f MiB | ms/step %.3f Mtok/s %.2f fwd %.3f ms | %s' % (L, NC, st_f32, st_bf16, d['ms_per_step'], d['value']/1e6, d['fwd']['ms_per_step'], ks))"
done; done
