#!/bin/bash
# final round-2 evidence on the final code: default bench (C2), reference arm, C3/C4/C5 lines, launch
# list, ncu full sets (C2 TTM + mTTV, C4 root mTTV), C2 PP timeline, Alg. 2 time to convergence
TAG=${TAG:-r2f}
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 6 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
for c in 3 4 5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c${c}_$TAG.log 2>&1; echo "config $c rc=$?"
done
CMD="python bench.py --steps 1 --warmup 1 --presweeps 2 --no-e2e --no-cpu-baseline --no-dmma-compare"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none -k regex:ttm_i8d -s 2 -c 1 -o /tmp/prof_ttm_$TAG $CMD > gpurun_out/ncu_ttm_$TAG.log 2>&1; echo "ncu ttm rc=$?"
ncu -i /tmp/prof_ttm_$TAG.ncu-rep --page raw --csv > gpurun_out/ttm_c2_$TAG.csv 2>/dev/null
ncu --set full --clock-control none -k regex:mttv_kernel -s 4 -c 1 -o /tmp/prof_mttv_$TAG $CMD > gpurun_out/ncu_mttv_$TAG.log 2>&1; echo "ncu mttv rc=$?"
ncu -i /tmp/prof_mttv_$TAG.ncu-rep --page raw --csv > gpurun_out/mttv_c2_$TAG.csv 2>/dev/null
C4="python bench.py --config 4 --steps 1 --warmup 1 --presweeps 0 --no-e2e --no-cpu-baseline --no-dmma-compare"
ncu --set full --clock-control none -k regex:mttv_kernel -c 1 -o /tmp/prof_c4m_$TAG $C4 > gpurun_out/ncu_c4m_$TAG.log 2>&1; echo "ncu c4 mttv rc=$?"
ncu -i /tmp/prof_c4m_$TAG.ncu-rep --page raw --csv > gpurun_out/mttv_c4_$TAG.csv 2>/dev/null
timeout 300 python tools/pp_timeline.py 2 > gpurun_out/pp_timeline_c2_$TAG.txt 2>&1; echo "timeline rc=$?"
for c in 2 4; do timeout 900 python tools/alg2_run.py $c 60 1e-5 any > gpurun_out/alg2_c${c}_$TAG.jsonl 2>&1; echo "alg2 c$c rc=$?"; done
