#!/bin/bash
# A/B of library variants on the exact-KL bench (run on the GPU box).
# usage: bash tools/ab_kl.sh base klold ...
mkdir -p gpurun_out
for i in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then unset RF_LIB_VARIANT; else export RF_LIB_VARIANT=$v; fi
    timeout 300 python bench.py --workload c2 --check 0 --kl-weight 0.1 --no-e2e --no-cpu-baseline --pool-gb 40 --steps 3 --warmup 2 \
      > gpurun_out/abkl_${v}_$i.log 2>&1
    echo "$v $i rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/abkl_${v}_$i.log | head -1)" >> gpurun_out/abkl_summary.txt
  done
done
unset RF_LIB_VARIANT
