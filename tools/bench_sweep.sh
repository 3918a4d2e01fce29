#!/bin/bash
# Filter-path tuning sweep: env knob settings -> per-kernel times.
# usage: bench_sweep.sh "VAR=a VAR2=b" "VAR=c" ...
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pk=d['roofline']['per_kernel']
print('ms_per_step %.4f e2e %.3f' % (d['ms_per_step'], d['e2e']['ms_per_step']))
for k,v in pk.items():
    print('  ', k, v if not isinstance(v, dict) else {x: (round(y,4) if isinstance(y,float) else y) for x,y in v.items() if x in ('ms','gbs','candidates')})
"
done
