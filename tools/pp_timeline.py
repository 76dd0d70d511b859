"""Back-to-back PP-approximated sweeps on a BASELINE config under CUPTI (torch.profiler): every
kernel of 4 consecutive pp_approx_sweep calls (no synchronisation between the calls, as in bench.py),
with its stream, start offset and duration (us), and the host time per call.  Shows the gaps on the
main stream between sweeps.  usage: python tools/pp_timeline.py [config] [max presweeps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2010_12056_b200 as cpd  # noqa: E402
import synth  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pres = int(sys.argv[2]) if len(sys.argv) > 2 else 60
cfg = synth.config(c)
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    T = bench.make_slab(cpd, torch, cfg, 0, 1, stream)
torch.cuda.synchronize()
m = cpd.cp_als_init(T, cfg.shape, cfg.R, synth.init_factors(cfg), stream=stream, pp_eps=0.2 if c == 4 else 0.1)
for _ in range(pres):  # until the PP entry condition holds (Alg. 2 line 5), as bench.py does
    m.msdt_sweep()
    if m.pp_condition():
        break
m.pp_init()
WARM = int(os.environ.get("WARM", "3"))      # untimed approximated sweeps after pp_init
PROF = int(os.environ.get("PROF", "4"))      # profiled back-to-back sweeps (C3: forced sweeps past the
for _ in range(WARM):                        # ε regime diverge on its structureless tensor; use 1 + 2)
    m.pp_approx_sweep()
torch.cuda.synchronize()
host = []
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(PROF):
        t0 = time.perf_counter()
        m.pp_approx_sweep()
        host.append(1e6 * (time.perf_counter() - t0))
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
g0 = evs[0].time_range.start
print("host us per call:", " ".join(f"{h:.0f}" for h in host))
print(f"gpu span {max(e.time_range.end for e in evs) - g0:.0f} us for {PROF} sweeps")
for e in evs:
    nm = e.name.replace("cpd::(anonymous namespace)::", "").replace("void ", "")[:44]
    print(f"{e.time_range.start - g0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  s{getattr(e, 'device_resource_id', '?')}  {nm}")
m.close()
