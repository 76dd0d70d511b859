#!/bin/bash
# ncu --set full captures of the first-level TTMs (every contraction position of one MSDT cycle)
# and the mTTV on C3, C4, C5, after a plain run of the same command exits 0.
# The .ncu-rep files are reduced to their raw-page CSV on the box (gpurun_out/ is capped at 64 MiB).
TAG=${TAG:-r2a}
mkdir -p gpurun_out
for c in ${CONFIGS:-3 4 5}; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --presweeps 0 --no-e2e --no-cpu-baseline --no-dmma-compare"
  timeout 600 $CMD > gpurun_out/plain_c${c}_$TAG.log 2>&1; echo "c$c plain rc=$?"
  tail -c 300 gpurun_out/plain_c${c}_$TAG.log
  NT=$(python -c "print({2:3,3:4,4:5,5:3}[$c])")
  timeout 1200 ncu --set full --clock-control none ${NCU_EXTRA} -k regex:${KREGEX:-ttm_i8d} -c $NT -o /tmp/ttm_c${c}_$TAG $CMD > gpurun_out/ncu_ttm_c${c}_$TAG.log 2>&1; echo "c$c ttm ncu rc=$?"
  ncu -i /tmp/ttm_c${c}_$TAG.ncu-rep --page raw --csv > gpurun_out/ttm_c${c}_$TAG.csv 2>/dev/null
  if [ -z "$NO_MTTV" ]; then
    timeout 600 ncu --set full --clock-control none -k regex:mttv_kernel -s 2 -c 2 -o /tmp/mttv_c${c}_$TAG $CMD > gpurun_out/ncu_mttv_c${c}_$TAG.log 2>&1; echo "c$c mttv ncu rc=$?"
    ncu -i /tmp/mttv_c${c}_$TAG.ncu-rep --page raw --csv > gpurun_out/mttv_c${c}_$TAG.csv 2>/dev/null
  fi
done
ls -la gpurun_out
