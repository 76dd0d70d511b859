timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "i8 or c1_full or order_N" > gpurun_out/t_i8.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/t_i8.log; grep -E "^E .*(Error|assert)" gpurun_out/t_i8.log | head -5
DBGS="0" bash tools/i8dbg.sh
timeout 300 python bench.py --ttm-impl int8 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_i8.log 2>&1; echo bench rc=$?
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench_i8.log').read().strip().splitlines()[-1])
print(d['value'], d['sweeps_ms'], d['roofline'])
PY
