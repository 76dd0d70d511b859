#!/bin/bash
# mTTV K-split target (waves) on C2 / C3 / C4 sweeps
for c in 2 3 4; do for w in 8 2 1; do
  CPD_MTTV_WAVES=$w timeout 300 python bench.py --config $c --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('c$c waves=$w'.ljust(20), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), 'stream frac %.3f' % d['roofline_stream']['frac'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
