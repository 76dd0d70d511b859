#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_shapes.py -q -x -p no:cacheprovider -k "i8 or dataset or full_size_sampled_rows or random" > gpurun_out/t14.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t14.log
for cfg in "" "CPD_I8_NO_MCF=1"; do env $cfg SHAPES="200,4,100" DBGS="0" timeout 600 bash tools/i8d_exp.sh 2>&1 | sed "s/^/[$cfg] /"; done
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > /tmp/b.log 2>&1
python -c "
import json;d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); s=d['sweeps_ms']; print('c3', 'msdt %.3f pp %.3f ppinit %.3f dt %.3f' % (s['msdt'], s['pp_approx'], s['pp_init'], s['dt']), d['roofline']['frac'], d['clocks']['sm_mhz'])"
