#!/bin/bash
# dual kernel at 512 threads / 64 registers, filler-stream mTTV at 3 CTAs/SM: PP tests, A/B benches
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_driver.py tests/test_gpu_random_shapes.py -q -x -p no:cacheprovider -k "pp or driver or random" > gpurun_out/t9.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t9.log
for rep in 1 2; do for cfg in "" "CPD_FILLER_OCC4=1"; do
  env $cfg timeout 300 python bench.py --config 2 --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('c2 [$cfg]'.ljust(26), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), d['clocks']['sm_mhz'])"
done; done
for c in 3 4; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('c$c'.ljust(26), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), d['clocks']['sm_mhz'])"
done
