#!/bin/bash
# PP sweep changes (speculative mode 0, fresh-init shortcut, main-stream stream ledger): PP parity
# tests, back-to-back PP timeline on C2, bench C2
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_driver.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "pp or c1 or driver or last_sweep or grid or fused or local_group" > gpurun_out/pptests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pptests.log
timeout 300 python tools/pp_timeline.py 2 > gpurun_out/pp_timeline_c2.txt 2>&1; echo "timeline rc=$?"; head -3 gpurun_out/pp_timeline_c2.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/bench_c2.log') if l.startswith('{')][-1]); print(d['value'], d['sweeps_ms'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline_stream'])"
SHAPES="200,4,100 2048,3,200" DBGS="0 33" timeout 900 bash tools/i8d_exp.sh 2>&1
