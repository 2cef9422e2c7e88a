#!/bin/bash
# Usage (on the GPU box, from the repo root): bash profiles/run_ncu.sh <tag> [kernel-regex] [extra bench args...]
# 1) plain run of the profiled command (must exit 0),
# 2) launch list of the TIMED region only (NVTX range "timed" in bench.py),
# 3) --set full on one launch of the kernel inside the timed region.
TAG=${1:-r01}
KREGEX=${2:-ring}
shift 2 2>/dev/null
CMD="python bench.py --steps 1 --warmup 1 --prompts 32 --no-e2e --no-cpu-baseline --check 0 --pool-gb 8 $*"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:$KREGEX -c 1 \
    -o gpurun_out/${TAG}_ring $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
# 4) SM->L2 store path and L2/DRAM traffic of the same launch (the write phase's bound)
ncu --nvtx --nvtx-include "timed/" --clock-control none -k regex:$KREGEX -c 1 --csv \
    --metrics gpu__time_duration.sum,l1tex__m_l1tex2xbar_write_bytes.sum,l1tex__m_l1tex2xbar_write_bytes.sum.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
    --log-file gpurun_out/${TAG}_storepath.csv $CMD > gpurun_out/${TAG}_ncu_store.log 2>&1
echo done
