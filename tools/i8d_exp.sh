#!/bin/bash
# int8 digit TTM: kernel-only durations (ncu gpu__time_duration) per mode for BASELINE shapes
# under the profiling switches CPD_I8_DBG (1 no MMA, 2 no loads, 4 no B loads, 8 no A loads, 32 no epilogue body)
for sh in ${SHAPES:-1024,3,64 200,4,100 64,5,32}; do
  shape=${sh//,/ }
  for d in ${DBGS:-0 1 2 32 35}; do
    CPD_I8_DBG=$d ONLY=int8 timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:ttm_i8d --csv python tools/prof_ttm_i8.py $shape 2>/dev/null \
     | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10 and r[-3]=='gpu__time_duration.sum']
v=[float(r[-1]) for r in rows]; u=rows[0][-2] if rows else ''
print('$shape dbg=$d', u, ' '.join('%.0f'%x for x in v), flush=True)"
  done
done
