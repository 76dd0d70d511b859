# bench lines for the other BASELINE configs (parity cases elsewhere); default N=1
for c in ${CONFIGS:-3 4 5}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-e2e --no-cpu-baseline ${EXTRA} > gpurun_out/bench_c$c.log 2>&1
  echo "config $c rc=$?"
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads([l for l in open(f'gpurun_out/bench_c{c}.log') if l.startswith('{')][-1])
    print(c, d['ttm_engine'], 'msdt', round(d['value'], 3), {k: round(v, 3) for k, v in d['sweeps_ms'].items()},
          'ttm', round(d['roofline']['avg_launch_ms'], 3), 'engines', json.dumps(d.get('engines'))[:400])
except Exception as e:
    print(c, 'no line', e, open(f'gpurun_out/bench_c{c}.log').read()[-1500:])
PY
done
