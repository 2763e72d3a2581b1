#!/bin/bash
# quick kernel-throughput comparison: each arg = "config n lanes block_threads block_sync [ik_iters]"
for spec in "$@"; do
  set -- $spec
  IK=${6:-0}
  python bench.py --config $1 --n $2 --lanes $3 --block-threads $4 --block-sync $5 --ik-iters $IK --steps 3 --warmup 2 --no-e2e --no-ttfs --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); c=d['config']; print('cfg',$1,'n',$2,'ik',$IK,'lanes',c['lanes_per_particle'],'threads',c['block_threads'],'bsync',c['block_sync'],'value %.3e'%d['value'],'kernel %.3e'%d['kernel_particle_steps_per_s'],'frac %.3f'%d['roofline']['frac'])
except Exception as e: print('FAIL',$1,$2,$3,$4,$5,l[-400:])
"
done
