#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --config 4 --steps 1 --warmup 1 --presweeps 0 --no-e2e --no-cpu-baseline --no-dmma-compare"
timeout 900 ncu --set full --clock-control none -k regex:mttv_kernel -c 14 -o /tmp/c4m $CMD > gpurun_out/ncu_c4m.log 2>&1; echo "rc=$?"
ncu -i /tmp/c4m.ncu-rep --page raw --csv > gpurun_out/mttv_c4_all.csv 2>/dev/null
