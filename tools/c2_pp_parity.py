"""C2 PP parity at full size ("after that, state-synchronised (incl. PP regime,
ε = 0.1)"): the GPU runs MSDT sweeps from the seeded factors until the PP condition holds, then
pp_init and `pp` approximated sweeps (the path bench.py times: operator streams on the filler
stream, the speculative next-sweep streams, the fused update with the V term).  The oracle builds
its own PP state from the GPU's factors at pp_init (Eq. 4 with explicit partial Khatri-Rao
products) and runs the same number of approximated sweeps from them (Eqs. 5-8): the fitness of
every sweep (tolerance 1e-10) and the final factors and M~^(n) are compared.
usage: python tools/c2_pp_parity.py [pp_sweeps] [config] -> one JSON line (config 2 by default; ε = 0.2 for C4)"""
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

npp = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = synth.config(c)
eps = 0.2 if c == 4 else 0.1
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    T = bench.make_slab(cpd, torch, cfg, 0, 1, stream)
torch.cuda.synchronize()
m = cpd.cp_als_init(T, cfg.shape, cfg.R, synth.init_factors(cfg), stream=stream, pp_eps=eps)
pre = 0
while pre < 60:
    m.msdt_sweep()
    pre += 1
    if m.pp_condition():
        break
A_init = [m.get_factor(n) for n in range(cfg.N)]
m.pp_init()
# back-to-back approximated sweeps with no other call in between, so the filler-stream
# speculation (the next sweep's mode-1 streams) is exercised; factors and M~ read at the end
f_gpu = [m.pp_approx_sweep() for _ in range(npp)]
A_end = [m.get_factor(n) for n in range(cfg.N)]
M_end = [m.get_last_mttkrp(n) for n in range(cfg.N)]
m.close()
del T
torch.cuda.empty_cache()

t0 = time.time()
To = O.make_tensor(cfg)
nt2 = O.norm2(To)
st = O.pp_init(To, A_init)
rows = []
A = A_init
for k in range(npp):
    out = O.pp_approx_sweep(st, A, nt2, eps)   # the oracle's own trajectory from A_init
    A = out["A"]
    f, valid = f_gpu[k]
    row = {"pp_sweep": k + 1, "f_gpu": f, "f_oracle": out["f"], "rel_df": abs(f - out["f"]) / abs(out["f"]),
           "still_valid": [int(valid), int(out["still_valid"])]}
    if k == npp - 1:
        row["rel_dA"] = [float(np.linalg.norm(A_end[n] - A[n]) / np.linalg.norm(A[n])) for n in range(cfg.N)]
        row["rel_dM"] = [float(np.linalg.norm(M_end[n] - out["M"][n]) / np.linalg.norm(out["M"][n]))
                         for n in range(cfg.N)]
    rows.append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
print(json.dumps({"config": cfg.name, "presweeps": pre, "pp_sweeps": npp, "tolerance": 1e-10,
                  "max_rel_df": max(r["rel_df"] for r in rows), "final_rel_dA": max(rows[-1]["rel_dA"]),
                  "final_rel_dM": max(rows[-1]["rel_dM"]),
                  "pass": all(r["rel_df"] <= 1e-10 for r in rows) and max(rows[-1]["rel_dM"]) <= 1e-10,
                  "oracle_s": time.time() - t0, "per_sweep": rows}))
