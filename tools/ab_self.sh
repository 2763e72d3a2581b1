for v in main slist main slist; do
  if [ $v = main ]; then L=""; else L="--lib exp/$v/libtamp.so"; fi
  timeout 300 python bench.py $L --config 3 --self-collision --steps 5 --warmup 3 --no-e2e --no-ttfs --no-cpu-baseline --no-extra 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('self $v', '%.4g' % d['value'], '%.4f ms' % d['kernel_ms_per_launch'], 'frac %.3f' % d['roofline']['frac'], d['config']['block_threads'])"
done
