#!/bin/bash
# Usage (on the GPU box, from the repo root): bash profiles/run_ncu.sh <tag> [kernel-regex] [extra bench args...]
# 1) plain run of the profiled command (must exit 0),
# 2) launch list of the TIMED region only (NVTX range "timed" in bench.py),
# 3) --set full on one launch of the kernel inside the timed region.
TAG=${1:-r01}
KREGEX=${2:-ring}
shift 2 2>/dev/null
CMD="python bench.py --steps 1 --warmup 1 --prompts 32 --no-e2e --no-cpu-baseline --pool-gb 8 $*"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:$KREGEX -c 1 \
    -o gpurun_out/${TAG}_ring $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
