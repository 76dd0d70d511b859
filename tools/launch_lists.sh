#!/bin/bash
# ncu launch lists (gpu__time_duration per launch) of bench.py on several configs
mkdir -p gpurun_out
for c in ${CONFIGS:-3 4}; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --presweeps 1 --no-e2e --no-cpu-baseline --no-dmma-compare"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c$c.csv $CMD > gpurun_out/ncu_list_c$c.log 2>&1
  echo "config $c ncu rc=$?"
  python tools/launch_summary.py gpurun_out/launches_c$c.csv | head -12
done
