#!/bin/bash
# A/B of environment settings on the C2 bench (run on the GPU box), interleaved twice.
# usage: bash tools/ab_env.sh "NAME1:ENV=VAL ENV2=VAL" "NAME2:" ...
mkdir -p gpurun_out
for i in 1 2; do
  for spec in "$@"; do
    name=${spec%%:*}; envs=${spec#*:}
    env $envs timeout 300 python bench.py --workload c2 --check 0 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 ${BENCH_ARGS} \
      > gpurun_out/abenv_${name}_$i.log 2>&1
    echo "$name $i rc=$? $(grep -o '"value": [0-9.]*' gpurun_out/abenv_${name}_$i.log | head -1)" >> gpurun_out/abenv_summary.txt
  done
done
