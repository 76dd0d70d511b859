#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_driver.py tests/test_gpu_random_shapes.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "not full_size and not dataset and not c2_full" > gpurun_out/t13.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t13.log
for cfg in "" "CPD_NO_LOCAL_INV=1"; do for c in 4 1; do
  env $cfg timeout 300 python bench.py --config $c --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('c$c [$cfg]'.ljust(28), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), d['clocks']['sm_mhz'])"
done; done
timeout 300 python tools/pp_timeline.py 4 3 > gpurun_out/pp_timeline_c4_local.txt 2>&1; sed -n 3,4p gpurun_out/pp_timeline_c4_local.txt
