#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "full_size_pp or large_rank or grid_validation" > gpurun_out/t11.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t11.log
