#!/bin/bash
# A/B: mTTV at 3 vs 4 resident CTAs per SM on C2 / C3 (alternating builds, same box)
for rep in 1 2 3; do for v in lb3 lb4; do
  cp build/ab/libcpd_$v.so paper_2010_12056_b200/libcpd.so
  timeout 300 python bench.py --config 2 --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('$v c2'.ljust(10), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), 'stream %.3f' % d['roofline_stream']['frac'], d['clocks']['sm_mhz'])"
done; done
