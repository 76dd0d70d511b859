"""Upper-level fusion on a BASELINE config: `python tools/msdt_levels_run.py c l [sweeps]` runs
msdt_sweep with opts.msdt_levels = l on the seeded config c (one MSDT cycle = N roots by default) and
prints the per-sweep device time, the roots ledger and cpd_get_memory (used under ncu for the launch
list of the block contractions)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_12056_b200 as cpd  # noqa: E402
import synth  # noqa: E402

c, l = int(sys.argv[1]), int(sys.argv[2])
cfg = synth.config(c)
n_sw = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.N - l
cpd.load_library()
T = torch.empty(cfg.shape, dtype=torch.float64, device="cuda")
if cfg.kind == "uniform":
    cpd.cpd_gen_tensor(T, cfg.shape, 0, cfg.s, 1, None, 0.0, cfg.seed_noise)
else:
    cpd.cpd_gen_tensor(T, cfg.shape, 0, cfg.s, 0, synth.true_factors(cfg), np.sqrt(cfg.noise_var), cfg.seed_noise)
m = cpd.cp_als_init(T, cfg.shape, cfg.R, synth.init_factors(cfg), msdt_levels=l)
m.msdt_sweep()
m.reset_counters()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
f = [m.msdt_sweep() for _ in range(n_sw)]
e1.record()
torch.cuda.synchronize()
print(json.dumps({"config": c, "msdt_levels": l, "sweeps": n_sw, "ms_per_sweep": e0.elapsed_time(e1) / n_sw,
                  "roots": m.counters()["roots"], "memory": m.get_memory(), "fitness": f[-1]}))
m.close()
