#!/bin/bash
# Launch-configuration sweep of bench.py on one config (GPU box).  Usage: bash tools/sweep_cfg.sh TAG CFG "lanes:threads:bsync ..." [extra bench args]
TAG=$1; CFG=$2; LIST=$3; shift 3
OUT=gpurun_out/sweep_$TAG.txt
: > $OUT
for item in $LIST; do
  IFS=: read L T S <<< "$item"
  line=$(timeout 300 python bench.py ${LIB:+--lib $LIB} --config $CFG --steps 5 --warmup 3 --no-e2e --no-ttfs --no-cpu-baseline --no-extra \
         --lanes $L --block-threads $T --block-sync $S "$@" 2>/dev/null | grep '^{')
  python - "$item" "$line" >> $OUT <<'PY'
import json, sys
item, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    print(f"{item:14s} value {d['value']:.4g}  K2 {d['kernel_particle_steps_per_s']:.4g}  frac {d['roofline']['frac']:.3f}  "
          f"ms/launch {d['kernel_ms_per_launch']:.4f}  threads {d['config']['block_threads']} lanes {d['config']['lanes_per_particle']}")
except Exception as e:
    print(f"{item:14s} FAILED {e}")
PY
done
cat $OUT
