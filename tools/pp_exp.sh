#!/bin/bash
# PP-approx sweep time (bench C2) under the update-grid cap and the mTTV K-split cap switches
for cfg in "" "CPD_UPD_BLOCKS=64" "CPD_UPD_BLOCKS=32" "CPD_UPD_BLOCKS=16" "CPD_MTTV_MAXKS=1" "CPD_MTTV_MAXKS=2" "CPD_UPD_BLOCKS=32 CPD_MTTV_MAXKS=1" "CPD_NO_PP_SPEC0=1"; do
  env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('$cfg'.ljust(40), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
