#!/bin/bash
# A/B of library variants (exp/<name>/libtamp.so) against the in-tree build: short bench lines per config.
# Usage: bash tools/ab_lib.sh "3 4 2" variant1 variant2 ...
CFGS=$1; shift
for cfg in $CFGS; do
  for v in main "$@" main; do
    if [ $v = main ]; then L=""; else L="--lib exp/$v/libtamp.so"; fi
    timeout 300 python bench.py $L --config $cfg --steps 5 --warmup 3 --no-e2e --no-ttfs --no-cpu-baseline --no-extra 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $cfg $v', '%.4g' % d['value'], '%.4f ms' % d['kernel_ms_per_launch'], 'frac %.3f' % d['roofline']['frac'], d['config']['block_threads'])"
  done
done
