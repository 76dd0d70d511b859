"""C2 full-trajectory parity (SURVEY §8(d) run schedule: "full trajectory for the first 6 MSDT
sweeps"): the GPU runs 6 msdt_sweep on the full 1024^3 tensor from the seeded initial factors;
the CPU oracle (explicit unfolding + explicit Khatri-Rao product + Cholesky, oracle.als_sweep)
runs 6 exact ALS sweeps from the same factors on its own copy of the tensor.  Per sweep: the
relative fitness difference (tolerance 1e-10) and the norm-wise factor differences.  Too long for
the pytest suite (the oracle needs ~30 s per sweep and ~30 GB of host memory), so it is a tool
whose output is committed under profiles/.
usage: python tools/c2_trajectory_parity.py [sweeps] -> one JSON line"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle as O  # noqa: E402
import paper_2010_12056_b200 as cpd  # noqa: E402
import synth  # noqa: E402

sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cfg = synth.config(2)
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    T = bench.make_slab(cpd, torch, cfg, 0, 1, stream)
torch.cuda.synchronize()
A0 = synth.init_factors(cfg)
m = cpd.cp_als_init(T, cfg.shape, cfg.R, A0, stream=stream)
f_gpu, A_gpu = [], []
for _ in range(sweeps):
    f_gpu.append(m.msdt_sweep())
    A_gpu.append([m.get_factor(n) for n in range(cfg.N)])
engine = m.ttm_engine()
m.close()
del T
torch.cuda.empty_cache()

t0 = time.time()
To = O.make_tensor(cfg)
nt2 = O.norm2(To)
A = A0
rows = []
for k in range(sweeps):
    out = O.als_sweep(To, A, nt2)
    A = out["A"]
    df = abs(f_gpu[k] - out["f"]) / abs(out["f"])
    dA = [float(np.linalg.norm(A_gpu[k][n] - A[n]) / np.linalg.norm(A[n])) for n in range(cfg.N)]
    rows.append({"sweep": k + 1, "f_gpu": f_gpu[k], "f_oracle": out["f"], "rel_df": df, "rel_dA": dA})
    print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
print(json.dumps({"config": "C2", "sweeps": sweeps, "ttm_engine": engine, "tolerance": 1e-10,
                  "max_rel_df": max(r["rel_df"] for r in rows),
                  "max_rel_dA": max(max(r["rel_dA"]) for r in rows),
                  "pass": all(r["rel_df"] <= 1e-10 for r in rows), "oracle_s": time.time() - t0,
                  "per_sweep": rows}))
