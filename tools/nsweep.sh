#!/bin/bash
# particle-count sweep (BASELINE config 5 shape): bench value / kernel rate / TTFS per N on one GPU
CFG=${1:-5}; shift
for N in "$@"; do
  python bench.py --config $CFG --n $N --steps 3 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline --no-extra 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); c=d['config']; t=d['ttfs']
  print('cfg',$CFG,'n',$N,'lanes',c['lanes_per_particle'],'threads',c['block_threads'],'value %.3e'%d['value'],'kernel %.3e'%d['kernel_particle_steps_per_s'],'frac %.3f'%d['roofline']['frac'],'ms_per_step %.2f'%d['ms_per_step'],'ttfs_s',t['s'],'ttfs_steps',t['steps'])
except Exception as e: print('FAIL',$CFG,$N,l[-300:])
"
done
