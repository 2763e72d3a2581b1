#!/bin/bash
# like profile.sh but for any kernel-name regex and extra bench args:  bash tools/profile_k.sh TAG REGEX [bench args...]
set -u
TAG=$1; RX=$2; shift 2
CMD="python bench.py --steps 2 --warmup 1 --repeats 1 --no-e2e --no-ttfs --no-cpu-baseline --no-extra $@"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$RX" -s 2 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "profile done"
