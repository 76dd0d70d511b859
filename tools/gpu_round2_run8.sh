#!/bin/bash
# mTTV at 64 registers (4 CTAs/SM) + packed narrow rows: full GPU suite incl. randomised shapes,
# bench C2/C3/C4 (C4 also without packing), C4 timeline
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1500 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gpu_tests.log
for c in 2 3 4; do
  timeout 300 python bench.py --config $c --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('c$c'.ljust(12), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), 'stream %.3f' % d['roofline_stream']['frac'], d['clocks']['sm_mhz'])"
done
CPD_MTTV_NO_PACK=1 timeout 300 python bench.py --config 4 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('c4 nopack'.ljust(12), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), 'stream %.3f' % d['roofline_stream']['frac'], d['clocks']['sm_mhz'])"
timeout 300 python tools/timeline.py 4 3 > gpurun_out/timeline_c4.txt 2>&1
