#!/bin/bash
# the round's evidence: default bench line, reference arm, per-config lines, launch list and ncu full sets
TAG=${1:-r06}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
bash tools/profile_run.sh $TAG
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"update_fused|gamma_inverse" -s 20 -c 2 -o gpurun_out/prof_small_$TAG python bench.py --steps 1 --warmup 1 --presweeps 2 --no-e2e --no-cpu-baseline --no-dmma-compare > gpurun_out/ncu_small_$TAG.log 2>&1; echo "small rc=$?"
CONFIGS="3 4 5" STEPS=3 bash tools/bench_configs.sh
