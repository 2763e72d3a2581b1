#!/bin/bash
# quick kernel-throughput comparison (no e2e / ttfs / cpu baseline)
for spec in "$@"; do
  set -- $spec
  python bench.py --config $1 --n $2 --lanes $3 --steps 3 --warmup 2 --no-e2e --no-ttfs --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('cfg',$1,'n',$2,'lanes',$3,'value %.3e'%d['value'],'kernel %.3e'%d['kernel_particle_steps_per_s'],'frac %.3f'%d['roofline']['frac'])
except Exception as e: print('FAIL',$1,$2,$3,l[-300:])
"
done
