timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
for v in main; do
  if [ $v = main ]; then L=""; else L="--lib exp/$v/libtamp.so"; fi
  timeout 300 python bench.py $L --config 1 --n 1048576 --steps 5 --warmup 3 --no-e2e --no-ttfs --no-cpu-baseline --no-extra 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['kernel_ms_per_launch'], d['roofline']['frac'], d['config']['block_threads'])"
done
