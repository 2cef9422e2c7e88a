#!/bin/bash
# All BASELINE.json configs on one GPU (run on the GPU box), each with the oracle check leg on
# 1,024 sampled rows of its last timed step: gpurun_out/sweep_<name>.log
mkdir -p gpurun_out
run() { name=$1; shift; timeout 1200 python bench.py --no-e2e --no-cpu-baseline --check 1024 "$@" > gpurun_out/sweep_$name.log 2>&1; echo "$name rc=$?" >> gpurun_out/sweep_rc.log; }
rm -f gpurun_out/sweep_rc.log
run c1 --workload c1 --steps 5 --warmup 3
run c2 --workload c2 --steps 5 --warmup 3
run c3_tis --workload c3 --variant tis --steps 3 --warmup 2
run c3_topr --workload c3 --variant topr --steps 3 --warmup 2
run c4 --workload c4 --steps 3 --warmup 2
run c5 --workload c5 --steps 3 --warmup 3
run c2_seqprod --workload c2 --aggregation sequence_product --steps 3 --warmup 2
run c2_kl --workload c2 --kl-weight 0.1 --steps 3 --warmup 2 --pool-gb 40
run c1_seqprod --workload c1 --aggregation sequence_product --steps 3 --warmup 2
run c2_ppo --workload c2 --variant ppo --steps 3 --warmup 2
run c2_cispo --workload c2 --variant cispo --steps 3 --warmup 2
run c2_grpo --workload c2 --variant grpo --steps 3 --warmup 2
run c2_naive_is --workload c2 --variant naive_is --steps 3 --warmup 2
