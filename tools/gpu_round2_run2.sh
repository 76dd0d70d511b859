#!/bin/bash
# digit-row padding experiment on the C3 TTM (KC / MCP boxes at 32-byte alignment), the new
# multirank tests (N-D grid, fused reduce-scatter), and the C3 / C4 bench lines
mkdir -p gpurun_out
python -c "import paper_2010_12056_b200 as p; p.load_library()"
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/multirank.log 2>&1; echo "multirank rc=$?"; tail -3 gpurun_out/multirank.log
for pad in 16 32 64; do
  CPD_DIGIT_PAD=$pad SHAPES="200,4,100" DBGS="0 1 33" timeout 600 bash tools/i8d_exp.sh 2>&1 | sed "s/^/pad=$pad /"
done
