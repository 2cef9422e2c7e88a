#!/bin/bash
# A/B of library variants on one box (run on the GPU box): interleaved C2 bench
# runs, each variant twice; results in gpurun_out/ab_<variant>_<i>.log.
# usage: bash tools/ab.sh base sup wf ...   ("base" = the default library)
mkdir -p gpurun_out
for i in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then unset RF_LIB_VARIANT; else export RF_LIB_VARIANT=$v; fi
    timeout 300 python bench.py --workload c2 --check 0 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ab_${v}_$i.log 2>&1
    echo "$v $i rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/ab_${v}_$i.log | head -1)" >> gpurun_out/ab_summary.txt
  done
done
unset RF_LIB_VARIANT
