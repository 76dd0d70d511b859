#!/bin/bash
# non-cooperative fused update (CPD_UPD_SPLIT) vs cooperative: parity subset under both, bench C2 x2
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
CPD_UPD_SPLIT=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_driver.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "not full_size and not dataset" > gpurun_out/split_tests.log 2>&1; echo "split tests rc=$?"; tail -2 gpurun_out/split_tests.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "full_size_sampled" > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?"; tail -2 gpurun_out/fullsize.log
for rep in 1 2; do for cfg in "" "CPD_UPD_SPLIT=1"; do
  env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
  python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('[$cfg]'.ljust(20), 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), d['clocks']['sm_mhz'])"
done; done
CPD_UPD_SPLIT=1 timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1; python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); print('c3 split', d['sweeps_ms'])"
