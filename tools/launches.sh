#!/bin/bash
# launch list (device time per kernel) of a short bench run with the given extra args; plain run first
TAG=$1; shift
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-ttfs --no-cpu-baseline $@"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo ok
