"""Time / profile the first-level TTM engines on a BASELINE shape (default C2: 1024^3, R=64).
usage: python tools/prof_ttm_i8.py [s N R] ; prints per-launch ms of DMMA and INT8 TTM per mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_12056_b200 as cpd  # noqa: E402

s, N, R = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 3, 64)
only = os.environ.get("ONLY", "")
cpd.load_library()
T = torch.randn([s] * N, dtype=torch.float64, device="cuda")
for j in range(N):
    A = torch.randn(s, R, dtype=torch.float64, device="cuda")
    pre, post = s ** j, s ** (N - 1 - j)
    out = torch.empty(pre * post, R, dtype=torch.float64, device="cuda")
    out2 = torch.empty_like(out)
    res = {}
    for name, fn in (("dmma", cpd.cpd_ttm), ("int8", cpd.cpd_ttm_i8)):
        if only and name != only:
            continue
        o = out if name == "dmma" else out2
        fn(T, pre, s, post, A, R, o)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn(T, pre, s, post, A, R, o)
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 3
    err = ((out - out2).norm() / out.norm()).item() if not only else float("nan")
    print(f"mode {j}: " + " ".join(f"{k} {v:.3f} ms" for k, v in res.items()) + f"  rel diff {err:.2e}", flush=True)
