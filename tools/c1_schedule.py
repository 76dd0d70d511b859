"""C1 whole-schedule latency (SURVEY §8(d) run schedule): from the seeded initial factors,
10 msdt_sweep, then pp_init + 5 forced pp_approx_sweep (reading Q14); 20 repeats on a fresh
context each (the first is a warm-up), median wall time of the blocking calls.  No roofline
claim: the 64^3 tensor (2 MB) is L2-resident and the schedule is launch/latency bound.
usage: python tools/c1_schedule.py [repeats]  -> one JSON line"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_12056_b200 as cpd  # noqa: E402
import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = synth.config(1)
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    T = bench.make_slab(cpd, torch, cfg, 0, 1, stream)
torch.cuda.synchronize()
A0 = synth.init_factors(cfg)
walls, fits = [], None
for rep in range(reps + 1):
    m = cpd.cp_als_init(T, cfg.shape, cfg.R, A0, stream=stream)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = [m.msdt_sweep() for _ in range(10)]
    m.pp_init()
    f += [m.pp_approx_sweep()[0] for _ in range(5)]
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    m.close()
    if rep > 0:
        walls.append(t1 - t0)
    fits = f
print(json.dumps({"config": "C1", "schedule": "10 msdt_sweep + pp_init + 5 pp_approx_sweep (forced)",
                  "repeats": reps, "median_ms": 1e3 * statistics.median(walls),
                  "min_ms": 1e3 * min(walls), "max_ms": 1e3 * max(walls),
                  "per_sweep_ms": 1e3 * statistics.median(walls) / 15, "final_fitness": fits[-1],
                  "fitness_trace": fits}))
