#!/bin/bash
# dual-output mTTV in the PP-init descent: operator parity tests (N = 3..8), full-size PP tests, PP-init times
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_driver.py -q -x -p no:cacheprovider -k "pp or grid or fused or driver or large_rank" > gpurun_out/dual_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/dual_tests.log
for c in 3 4 2; do for cfg in "" "CPD_PP_NO_DUAL=1"; do
  env $cfg timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('c$c [$cfg]'.ljust(26), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), d['clocks']['sm_mhz'])"
done; done
