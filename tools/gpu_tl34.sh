#!/bin/bash
mkdir -p gpurun_out
for c in 4 3; do timeout 300 python tools/pp_timeline.py $c 3 > gpurun_out/pp_timeline_c$c.txt 2>&1; echo "c$c rc=$?"; sed -n 3,4p gpurun_out/pp_timeline_c$c.txt; done
for c in 3 4; do CPD_NO_FUSED_UPDATE=1 timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('c$c nofused'.ljust(14), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), d['clocks']['sm_mhz'])"; done
