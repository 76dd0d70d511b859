DBGS="6 14 0" bash tools/i8dbg.sh
CPD_I8_DBG=6 ONLY=int8 ncu --set full --import-source on -k regex:ttm_i8_kernel -s 8 -c 1 -o gpurun_out/prof_i8_dbg6 python tools/prof_ttm_i8.py > /dev/null 2>&1
CPD_I8_DBG=0 ONLY=int8 ncu --set full --import-source on -k regex:ttm_i8_kernel -s 8 -c 1 -o gpurun_out/prof_i8_dbg0 python tools/prof_ttm_i8.py > /dev/null 2>&1
echo done
