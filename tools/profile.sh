#!/bin/bash
# Run on the GPU box (gpurun): plain bench first (must exit 0), then the ncu launch list and one full
# capture of the dominant kernel (k_particle<MODE_OPT>).  Output under gpurun_out/.
#   bash tools/profile.sh TAG CONFIG [N]
set -u
TAG=${1:-r1}
CFG=${2:-2}
N=${3:-0}
NARG=""
if [ "$N" != "0" ]; then NARG="--n $N"; fi
CMD="python bench.py --config $CFG $NARG --steps 2 --warmup 1 --repeats 1 --no-e2e --no-ttfs --no-cpu-baseline --no-extra"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_particle<.int.0," -s 2 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "profile done"
