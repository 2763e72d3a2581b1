#!/bin/bash
# A/B of library variants (exp/<name>/libtamp.so, tools/build_variants.py) against the in-tree build on the given
# configs (GPU box).  Usage: bash tools/ab_variants.sh "3 2 4" v1 v2 ...
CFGS=$1; shift
for cfg in $CFGS; do
  for v in main "$@"; do
    if [ $v = main ]; then L=""; else L=exp/$v/libtamp.so; fi
    LIB=$L bash tools/sweep_cfg.sh ab_${v}_$cfg $cfg "0:0:-1" > /dev/null 2>&1
    echo "cfg $cfg $v $(cat gpurun_out/sweep_ab_${v}_$cfg.txt)"
  done
done
