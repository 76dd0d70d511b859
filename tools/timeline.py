"""Kernel timeline (all streams, CUPTI via torch.profiler) of one MSDT cycle, pp_init and two
PP-approximated sweeps on a BASELINE config.  usage: python tools/timeline.py [config] [presweeps] [auto|dmma|int8]
Prints every kernel with its stream, start offset and duration (us), per sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2010_12056_b200 as cpd  # noqa: E402
import synth  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pres = int(sys.argv[2]) if len(sys.argv) > 2 else 5
impl = sys.argv[3] if len(sys.argv) > 3 else "auto"
cfg = synth.config(c)
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    T = bench.make_slab(cpd, torch, cfg, 0, 1, stream)
torch.cuda.synchronize()
m = cpd.cp_als_init(T, cfg.shape, cfg.R, synth.init_factors(cfg), stream=stream,
                    pp_eps=0.2 if c == 4 else 0.1, ttm_impl=bench.TTM_IMPL[impl])
for _ in range(pres):
    m.msdt_sweep()
m.pp_init()
m.pp_approx_sweep()
torch.cuda.synchronize()
marks = []
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for name, fn in [("msdt", m.msdt_sweep), ("msdt", m.msdt_sweep), ("pp_init", m.pp_init),
                     ("pp", m.pp_approx_sweep), ("pp", m.pp_approx_sweep)]:
        torch.cuda.synchronize()
        with torch.profiler.record_function("SWEEP_" + name):
            fn()
        torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
cpu_marks = sorted([e for e in prof.events() if e.name.startswith("SWEEP_")], key=lambda e: e.time_range.start)
kern = sorted(evs, key=lambda e: e.time_range.start)
for mk in cpu_marks:
    t0, t1 = mk.time_range.start, mk.time_range.end
    ks = [e for e in kern if t0 <= e.time_range.start <= t1]
    if not ks:
        continue
    g0 = ks[0].time_range.start
    gend = max(e.time_range.end for e in ks)
    busy = sum(e.time_range.end - e.time_range.start for e in ks)
    print(f"== {mk.name}: host {t1 - t0:.0f} us, gpu span {gend - g0:.0f} us, kernel-sum {busy:.0f} us, {len(ks)} kernels")
    for e in ks:
        nm = e.name.replace("cpd::(anonymous namespace)::", "").replace("void ", "")[:44]
        print(f"   {e.time_range.start - g0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  s{getattr(e, 'device_resource_id', '?')}  {nm}")
m.close()
