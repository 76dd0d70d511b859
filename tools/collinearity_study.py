"""Collinearity time-to-convergence study (the paper's Fig. 4 / Table 3,
P:819-853): order-3 exact CP tensors s x s x s whose factor columns have pairwise cosine C
(construction Q13), C drawn from [a, b) per bin with a seeded RNG; PP-CP-ALS
(Alg. 2, ε = 0.2, MSDT regular sweeps), MSDT ALS and DT ALS from the same U[0,1] initial
factors (Alg. 2 line 2), stopped at Δf <= 1e-5 between neighbouring sweeps or 300
sweeps.  The paper uses s = 1600, R = 400 on 64 KNL processes.
usage: python tools/collinearity_study.py [s] [R] [seeds] [max_sweeps] [any|regular]
(the Δ stop test: neighbouring sweeps of any kind, reading Q21, or consecutive regular sweeps
as Alg. 2 prints it) -> one JSON line per run"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2010_12056_b200 as cpd  # noqa: E402
import synth  # noqa: E402
from paper_2010_12056_b200.driver import phase_counts, pp_cp_als  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
R = int(sys.argv[2]) if len(sys.argv) > 2 else 200
seeds = int(sys.argv[3]) if len(sys.argv) > 3 else 1
max_sweeps = int(sys.argv[4]) if len(sys.argv) > 4 else 300
stop_test = sys.argv[5] if len(sys.argv) > 5 else "any"
stream = torch.cuda.Stream()
for b in range(5):
    lo, hi = 0.2 * b, 0.2 * (b + 1)
    for seed in range(seeds):
        C = float(np.random.default_rng(100 * b + seed).uniform(lo, hi))
        cfg = synth.custom(3, s, R, noise_var=0.0, collinearity=C, seed=500 + 10 * b + seed)
        with torch.cuda.stream(stream):
            T = bench.make_slab(cpd, torch, cfg, 0, 1, stream)
        torch.cuda.synchronize()
        g = np.random.default_rng(900 + 10 * b + seed)
        A0 = [g.random((s, R)) for _ in range(3)]           # U[0,1] (Alg. 2 line 2)
        res = {}
        for name, eps, regular in [("pp", 0.2, "msdt"), ("msdt", 1e-300, "msdt"), ("dt", 1e-300, "dt")]:
            m = cpd.cp_als_init(T, cfg.shape, R, A0, stream=stream, pp_eps=eps)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rows = pp_cp_als(m, delta=1e-5, max_sweeps=max_sweeps, regular=regular, stop_test=stop_test)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            fits = [r[3] for r in rows if r[3] is not None]
            res[name] = {"wall_s": wall, "counts": phase_counts(rows), "final_fitness": fits[-1]}
            m.close()
        print(json.dumps({"s": s, "R": R, "stop_test": stop_test, "bin": [round(lo, 1), round(hi, 1)], "C": C, "seed": seed,
                          "runs": res, "pp_speedup_vs_dt": res["dt"]["wall_s"] / res["pp"]["wall_s"],
                          "pp_speedup_vs_msdt": res["msdt"]["wall_s"] / res["pp"]["wall_s"],
                          "msdt_speedup_vs_dt": res["dt"]["wall_s"] / res["msdt"]["wall_s"]}), flush=True)
        del T
        torch.cuda.empty_cache()
