#!/bin/bash
# config 1 at 1M particles (serial mapping): tests + bench of the in-tree build and A/B library variants / flags.
# Usage: bash tools/ab_cfg1.sh [tests] ["label:extra bench args" ...]
if [ "$1" = tests ]; then shift; timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; tail -1 gpurun_out/gputests.log; fi
for spec in "main:" "$@"; do
  lab=${spec%%:*}; args=${spec#*:}
  timeout 300 python bench.py --config 1 --n 1048576 --steps 5 --warmup 3 --no-e2e --no-ttfs --no-cpu-baseline --no-extra $args 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', '%.4g' % d['value'], '%.4f ms' % d['kernel_ms_per_launch'], 'frac %.3f' % d['roofline']['frac'], d['config']['block_threads'], 'bsync', d['config']['block_sync'])"
done
