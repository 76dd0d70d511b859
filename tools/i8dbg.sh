# profiling switches of the int8 TTM (CPD_I8_DBG bits: 1 no MMA, 2 no loads, 4 no conversion)
# kernel-only durations from ncu (gpu__time_duration), modes 0,1,2 x 4 launches each
for d in ${DBGS:-0 1 2 4 6 3 5}; do
  CPD_I8_DBG=$d ONLY=int8 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:ttm_i8 --csv python tools/prof_ttm_i8.py 2>/dev/null \
   | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10 and r[-3]=='gpu__time_duration.sum']
v=[float(r[-1]) for r in rows]; u=rows[0][-2] if rows else ''
print('dbg=$d', u, ' '.join('%.0f'%x for x in v))"
done
