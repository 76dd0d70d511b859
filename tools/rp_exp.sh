#!/bin/bash
# N-tile width experiment for the digit TTM (CPD_I8_RPMAX 64 vs 32): kernel times + C2/C3 bench lines
for rp in 64 32; do
  CPD_I8_RPMAX=$rp DBGS=0 bash tools/i8d_exp.sh 2>&1 | sed "s/^/rpmax=$rp /"
done
for c in 2 3; do for rp in 64 32; do
  CPD_I8_RPMAX=$rp timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-dmma-compare > gpurun_out/bench_rp${rp}_c$c.log 2>&1
  python - $c $rp <<'PY'
import json, sys
c, rp = sys.argv[1:3]
try:
    d = json.loads([l for l in open(f'gpurun_out/bench_rp{rp}_c{c}.log') if l.startswith('{')][-1])
    print('config', c, 'rpmax', rp, {k: round(v, 3) for k, v in d['sweeps_ms'].items()}, 'ttm', round(d['roofline']['avg_launch_ms'], 3))
except Exception as e:
    print(c, rp, 'no line', e, open(f'gpurun_out/bench_rp{rp}_c{c}.log').read()[-1500:])
PY
done; done
