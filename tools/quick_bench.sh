#!/bin/bash
# GPU suite + short bench lines of the main workloads (value, kernel, frac).  Usage: bash tools/quick_bench.sh [tests]
if [ "$1" = tests ]; then timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; tail -1 gpurun_out/gputests.log; fi
for spec in "3 32768" "2 8192" "1 1048576" "4 16384"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --n $2 --steps 5 --warmup 3 --no-ttfs --no-cpu-baseline --no-extra 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('cfg $1 n $2 value %.4g e2e %.4g kernel %.4g ms/launch %.4f frac %.3f threads %s lanes %s' % (d['value'], d['e2e']['value'], d['kernel_particle_steps_per_s'], d['kernel_ms_per_launch'], d['roofline']['frac'], d['config']['block_threads'], d['config']['lanes_per_particle']))"
done
