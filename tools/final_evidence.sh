#!/bin/bash
# End-of-round evidence on one B200 (gpurun): GPU suite, bench lines, ncu launch lists and full captures of the hot
# kernels, the particle-count sweep.  Everything under gpurun_out/$TAG/.
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/gputests.log 2>&1; tail -3 $O/gputests.log
bash tools/device_checks.sh > $O/device_checks.log 2>&1; tail -1 $O/device_checks.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_default.log 2>&1
python bench.py --impl reference > $O/bench_reference.log 2>&1
python bench.py --config 2 --no-cpu-baseline --no-extra > $O/bench_cfg2.log 2>&1
python bench.py --config 1 --n 1048576 --no-cpu-baseline --no-extra > $O/bench_cfg1_1m.log 2>&1
python bench.py --config 4 --no-cpu-baseline --no-extra > $O/bench_cfg4.log 2>&1
bash tools/nsweep.sh 5 1024 4096 16384 65536 262144 1048576 > $O/nsweep_cfg5.txt 2>&1
bash tools/nsweep.sh 1 256 4096 65536 262144 1048576 > $O/nsweep_cfg1.txt 2>&1
CMD="python bench.py --steps 2 --warmup 1 --repeats 1 --no-e2e --no-ttfs --no-cpu-baseline --no-extra"
for c in 3 2; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg$c.csv $CMD --config $c > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_particle<.int.0," -s 2 -c 1 -o $O/prof_cfg$c $CMD --config $c > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg1_1m.csv $CMD --config 1 --n 1048576 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_serial<.int.0" -s 2 -c 1 -o $O/prof_cfg1_1m $CMD --config 1 --n 1048576 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_particle<.int.0," -s 2 -c 1 -o $O/prof_cfg4 $CMD --config 4 > /dev/null 2>&1
echo done
