"""Time to convergence on a BASELINE config (SURVEY §8(d) run schedule; the paper's Tables 3/4
and Figs. 5-6 compare the same three runs on CPU clusters):
  * PP-CP-ALS   Alg. 2 with MSDT regular sweeps, eps from the config,
  * MSDT ALS    plain CP-ALS on the multi-sweep dimension tree (the PP test never passes),
  * DT ALS      plain CP-ALS on the standard dimension tree,
all from the same seeded tensor and initial factors, stopping when the fitness of two
neighbouring sweeps differs by <= delta or after max_sweeps.
With LEVELS=l (environment, order >= 4) two more runs use upper-level fusion (msdt_levels = l,
P:700-702): PP-CP-ALS and MSDT ALS at that l.
usage: python tools/alg2_run.py [config] [max_sweeps] [delta] [any|regular]  -> one JSON line per run"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_12056_b200 as cpd  # noqa: E402
import synth  # noqa: E402
from paper_2010_12056_b200.driver import phase_counts, pp_cp_als  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
max_sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
delta = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-5
stop_test = sys.argv[4] if len(sys.argv) > 4 else "any"
cfg = synth.config(c)
eps = 0.2 if c == 4 else 0.1
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    T = bench.make_slab(cpd, torch, cfg, 0, 1, stream)
torch.cuda.synchronize()
A0 = synth.init_factors(cfg)
runs = [("pp_cp_als", {"pp_eps": eps}, "msdt"),
        ("msdt_als", {"pp_eps": 1e-300}, "msdt"),
        ("dt_als", {"pp_eps": 1e-300}, "dt")]
lv = int(os.environ.get("LEVELS", "1"))
if lv > 1:
    runs += [(f"pp_cp_als_l{lv}", {"pp_eps": eps, "msdt_levels": lv}, "msdt"),
             (f"msdt_als_l{lv}", {"pp_eps": 1e-300, "msdt_levels": lv}, "msdt")]
for name, kw, regular in runs:
    m = cpd.cp_als_init(T, cfg.shape, cfg.R, A0, stream=stream, **kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = pp_cp_als(m, delta=delta, max_sweeps=max_sweeps, regular=regular, stop_test=stop_test)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    per = {}
    for r in rows:
        per.setdefault(r[1], []).append(r[4])
    fits = [r[3] for r in rows if r[3] is not None]
    print(json.dumps({
        "config": cfg.name, "run": name, "stop_test": stop_test, "eps": kw["pp_eps"] if name.startswith("pp_cp_als") else None,
        "msdt_levels": kw.get("msdt_levels", 1), "delta": delta,
        "sweeps": len(fits), "phase_counts": phase_counts(rows), "wall_s": wall,
        "ms_per_phase": {k: 1e3 * sum(v) / len(v) for k, v in per.items()},
        "final_fitness": fits[-1] if fits else None, "ttm_engine": m.ttm_engine(),
        "fitness_trace": [round(f, 10) for f in fits[:: max(1, len(fits) // 40)]],
    }), flush=True)
    m.close()
