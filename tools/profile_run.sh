#!/bin/bash
# ncu evidence for the bench command (B200_PROFILING.md recipe): plain run, launch list, full sets
CMD="python bench.py --steps 1 --warmup 1 --presweeps 2 --no-e2e --no-cpu-baseline --no-dmma-compare"
TAG=${1:-r01}
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ttm_i8d -s 2 -c 1 -o gpurun_out/prof_ttm_$TAG $CMD > gpurun_out/ncu_ttm_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mttv_kernel -s 4 -c 1 -o gpurun_out/prof_mttv_$TAG $CMD > gpurun_out/ncu_mttv_$TAG.log 2>&1
echo "rc=$?"
