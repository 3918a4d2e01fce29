#!/bin/bash
# Filter-path tuning sweep: bins per chunk (log2) -> per-kernel times.
for b in 6 7 8; do
  echo "== bins/chunk 2^$b"
  CHGPU_FILTER_BINS_PER_CHUNK_LOG2=$b timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
pk=d['roofline']['per_kernel']
print('ms_per_step %.4f e2e %.3f' % (d['ms_per_step'], d['e2e']['ms_per_step']))
for k,v in pk.items():
    print('  ', k, v if not isinstance(v, dict) else {x: (round(y,4) if isinstance(y,float) else y) for x,y in v.items() if x in ('ms','gbs','candidates')})
"
done
