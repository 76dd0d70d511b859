#!/bin/bash
# final evidence of round 2 on the final code: GPU suite + smoke, bench lines (C2 default + reference arm,
# C3 / C4 at msdt_levels 1 and 2, C5), C2 launch list, ncu --set full of the first-level TTMs of one MSDT
# cycle on C2-C5 and of the C3 mTTV (traffic per launch for bench.py's roofline), C2 PP timeline
TAG=${TAG:-r2h}
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 6 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
for c in 3 4; do for l in 1 2; do
  timeout 900 python bench.py --config $c --msdt-levels $l --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c${c}_l${l}_$TAG.log 2>&1; echo "config $c l=$l rc=$?"
done; done
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_$TAG.log 2>&1; echo "config 5 rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --presweeps 2 --no-e2e --no-cpu-baseline --no-dmma-compare"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1; echo "launch list rc=$?"
for c in 2 3 4 5; do
  C="python bench.py --config $c --steps 1 --warmup 1 --presweeps 0 --no-e2e --no-cpu-baseline --no-dmma-compare"
  NT=$(python -c "print({2:3,3:4,4:5,5:3}[$c])")
  timeout 1200 ncu --set full --clock-control none -k regex:ttm_i8d -c $NT -o /tmp/ttm_c${c}_$TAG $C > gpurun_out/ncu_ttm_c${c}_$TAG.log 2>&1; echo "c$c ttm ncu rc=$?"
  ncu -i /tmp/ttm_c${c}_$TAG.ncu-rep --page raw --csv > gpurun_out/ttm_c${c}_$TAG.csv 2>/dev/null
done
C3="python bench.py --config 3 --steps 1 --warmup 1 --presweeps 0 --no-e2e --no-cpu-baseline --no-dmma-compare"
timeout 600 ncu --set full --clock-control none -k regex:mttv_kernel -s 2 -c 2 -o /tmp/mttv_c3_$TAG $C3 > gpurun_out/ncu_mttv_c3_$TAG.log 2>&1; echo "c3 mttv ncu rc=$?"
ncu -i /tmp/mttv_c3_$TAG.ncu-rep --page raw --csv > gpurun_out/mttv_c3_$TAG.csv 2>/dev/null
timeout 300 python tools/pp_timeline.py 2 > gpurun_out/pp_timeline_c2_$TAG.txt 2>&1; echo "timeline rc=$?"
ls -la gpurun_out | tail -40
