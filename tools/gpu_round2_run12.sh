#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "c2_full_trajectory or fused or grid or local_group" > gpurun_out/t12.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t12.log
