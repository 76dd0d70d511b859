#!/bin/bash
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()" 
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1500 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_default.log
SHAPES="200,4,100 64,5,32" DBGS="0 1 2 32 33" timeout 600 bash tools/i8d_exp.sh > gpurun_out/i8d_exp.log 2>&1; echo "exp rc=$?"
cat gpurun_out/i8d_exp.log
