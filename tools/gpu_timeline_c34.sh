#!/bin/bash
mkdir -p gpurun_out
for c in 4 3; do timeout 300 python tools/timeline.py $c 3 > gpurun_out/timeline_c$c.txt 2>&1; echo "c$c rc=$?"; done
