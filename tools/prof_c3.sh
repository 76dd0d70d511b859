#!/bin/bash
# full-set ncu capture of the four first-level TTMs of a C3 MSDT cycle (KC, MCP 4-D, MCP 5-D x2)
mkdir -p gpurun_out
C3="python bench.py --config 3 --steps 1 --warmup 1 --presweeps 0 --no-e2e --no-cpu-baseline --no-dmma-compare"
T=${TAG:-r06}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ttm_i8d -c 4 -o gpurun_out/c3_ttm_$T $C3 > gpurun_out/c3_ttm.log 2>&1; echo c3 ttm ncu $?
