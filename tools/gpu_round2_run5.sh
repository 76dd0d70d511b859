#!/bin/bash
# PP speculation fix + split mode-0 speculation: full GPU suite, C2 PP timeline, bench C2
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1500 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gpu_tests.log
timeout 300 python tools/pp_timeline.py 2 > gpurun_out/pp_timeline_c2.txt 2>&1; echo "timeline rc=$?"; sed -n 3,4p gpurun_out/pp_timeline_c2.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/bench_c2.log') if l.startswith('{')][-1]); print(d['value'], d['sweeps_ms'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline_stream']['frac'], d['pp_filler_streams'])"
