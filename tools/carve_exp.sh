#!/bin/bash
for rep in 1 2; do for cfg in "" "CPD_MTTV_CARVEOUT=1"; do
  env $cfg timeout 300 python bench.py --config 2 --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('[$cfg]'.ljust(24), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), d['clocks']['sm_mhz'])"
done; done
CPD_MTTV_CARVEOUT=1 timeout 300 python tools/pp_timeline.py 2 > gpurun_out/pp_timeline_carve.txt 2>&1; sed -n 3,4p gpurun_out/pp_timeline_carve.txt
