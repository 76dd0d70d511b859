#!/bin/bash
# W of Eq. 7 fused into the Γ^-1 launch: PP tests, smoke, C2/C4 PP timings
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_driver.py tests/test_gpu_random_shapes.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "pp or driver or random or grid or fused" > gpurun_out/t10.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t10.log
for c in 2 4; do
  timeout 300 python bench.py --config $c --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('c$c'.ljust(8), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), d['clocks']['sm_mhz'])"
done
