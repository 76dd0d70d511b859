#!/bin/bash
# digit TTM after the one-wait-per-chunk drain and the rotating multicast issuer: i8 parity tests,
# per-mode kernel times (C2, C3, C4 shapes), bench lines C2 and C3
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "i8 or c1_full or msdt_and_dt or pp_order" > gpurun_out/i8tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/i8tests.log
SHAPES="1024,3,64 200,4,100 64,5,32 2048,3,200" DBGS="0 33" timeout 900 bash tools/i8d_exp.sh 2>&1
for c in 2 3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench c$c rc=$?"; python -c "
import json;d=json.loads([l for l in open('gpurun_out/bench_c$c.log') if l.startswith('{')][-1]); print(d['value'], d['sweeps_ms'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline'].get('tensor_int8',{}).get('frac'), d['roofline_stream']['frac'])"; done
